// models.hpp — synthetic inputs, model builders and model-walk helpers (models.cpp).
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "sige_b200.h"

namespace sige_b200 {

constexpr uint64_t kFnvSeed = 1469598103934665603ull;
uint64_t fnv1a64(const void* data, size_t bytes, uint64_t seed = kFnvSeed);

void make_edit_fixture(const std::string& kind, int n, int c, int h, int w, uint32_t seed,
                       float* orig, float* edited);
sige_model_desc* build_model(const std::string& name);
// Config 3 inputs: one-hot segmentation map and its edit (a relabelled 1.2 % square).
void make_seg_fixture(int n, int label_nc, int h, int w, uint32_t seed, float* orig, float* edited);
void free_model(sige_model_desc* d);
uint64_t model_weight_hash(const sige_model_desc* d);
uint64_t model_structure_hash(const sige_model_desc* d);  // ModelSpec::structure_hash (graph.cpp:89-127)

struct LayerShape {
  int c_in, h_in, w_in, c_out, h_out, w_out;
};
std::vector<LayerShape> walk_shapes(const sige_model_desc* m);
int required_dilation(const sige_model_desc* m);

}  // namespace sige_b200
