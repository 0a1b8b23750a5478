// sige_b200.hpp — the reference-side C++ adapter over the C ABI (sige_b200.h).
//
// The reference (proj/include/sige/*.hpp) has no FFI: its sparse path is a
// value-semantics free-function API in namespace `sige`. This header restores
// exactly that API on top of libsige_b200 — same names, same argument types
// (sige::Tensor, DifferenceMask, BlockIndexSet, BlockStack, Epilogue,
// ConvLayer, ScatterMap, ModelSpec, RunConfig), results returned as fresh
// host values, sige::ConfigError for every ConfigError the library reports —
// so reference code switches path by qualifying calls with `sige::b200::`.
// Host values are staged through device buffers per call (the op-level
// functions are synchronous, like the reference's); the Engine keeps the
// model and its ActivationCache resident in HBM.
//
// Include after the reference headers' directory is on the include path
// (proj/include) and link libsige_b200.so (cudart static inside) plus cudart
// for the staging copies. tests/test_adapter.py compiles this header against
// /root/reference/proj/include and runs the reference's own acceptance
// criteria 1, 3 and 5 (proj/tests/acceptance.cpp:52-253, 306-330) through it
// (tests/native/adapter_acceptance.cpp).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sige/common.hpp"
#include "sige/conv.hpp"
#include "sige/eltwise.hpp"
#include "sige/graph.hpp"
#include "sige/kernels.hpp"
#include "sige/mask.hpp"
#include "sige/tensor.hpp"
#include "sige_b200.h"

namespace sige {
namespace b200 {

// ---- errors ---------------------------------------------------------------

inline void check(int rc) {  // SIGE_ERR_CONFIG -> sige::ConfigError (common.hpp:14-17)
  if (rc == SIGE_OK) return;
  if (rc == SIGE_ERR_CONFIG) throw ConfigError(sige_last_error());
  throw std::runtime_error(sige_last_error());
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- device staging ---------------------------------------------------------

template <class T>
class DevBuf {
 public:
  explicit DevBuf(size_t n) : n_(n) {
    cuda_check(cudaMalloc(&p_, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  }
  explicit DevBuf(const std::vector<T>& h) : DevBuf(h.size()) { upload(h.data(), h.size()); }
  DevBuf(const T* h, size_t n) : DevBuf(n) { upload(h, n); }
  ~DevBuf() { cudaFree(p_); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const T* h, size_t n) {
    if (n) cuda_check(cudaMemcpy(p_, h, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  }
  void download(T* h, size_t n) const {
    cuda_check(cudaDeviceSynchronize(), "kernel");
    if (n) cuda_check(cudaMemcpy(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  }
  std::vector<T> to_host() const {
    std::vector<T> h(n_);
    download(h.data(), n_);
    return h;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

inline DevBuf<int32_t> upload_indices(const BlockIndexSet& s) {  // BlockIndex {n, r, c} -> int32 triplets
  std::vector<int32_t> v;
  v.reserve(s.indices.size() * 3);
  for (const BlockIndex& b : s.indices) v.insert(v.end(), {b.n, b.r, b.c});
  return DevBuf<int32_t>(v);
}

inline BlockIndexSet download_indices(const int32_t* host, size_t count, int block, int h, int w) {
  BlockIndexSet s;
  s.block_size = block;
  s.h = h;
  s.w = w;
  s.indices.resize(count);
  for (size_t i = 0; i < count; ++i) s.indices[i] = {host[3 * i], host[3 * i + 1], host[3 * i + 2]};
  return s;
}

// sige::Epilogue (eltwise.hpp:30-59) -> sige_epilogue with device parameters.
class DevEpilogue {
 public:
  explicit DevEpilogue(const Epilogue& e) {
    if (e.steps.size() > SIGE_MAX_EPI_STEPS)
      throw ConfigError("epilogue: more than " + std::to_string(SIGE_MAX_EPI_STEPS) + " pending element-wise steps");
    c_.num_steps = static_cast<int>(e.steps.size());
    for (size_t k = 0; k < e.steps.size(); ++k) {
      const Epilogue::Step& s = e.steps[k];
      sige_epilogue_step& d = c_.steps[k];
      if (s.kind == Epilogue::Step::Kind::ScaleShift) {
        d.kind = SIGE_EPI_SCALE_SHIFT;
        d.nparams = static_cast<int>(s.scale.size());
        keep_.push_back(std::make_unique<DevBuf<float>>(s.scale));
        d.scale = keep_.back()->get();
        keep_.push_back(std::make_unique<DevBuf<float>>(s.shift));
        d.shift = keep_.back()->get();
      } else {
        d.kind = SIGE_EPI_ACTIVATION;
        d.act = static_cast<int>(s.act);  // ActKind {None, Relu, Silu} == SIGE_ACT_*
      }
    }
  }
  const sige_epilogue* get() const { return &c_; }

 private:
  sige_epilogue c_{};
  std::vector<std::unique_ptr<DevBuf<float>>> keep_;
};

// sige::ConvLayer (conv.hpp:11-23) with device weights (op-level calls).
class DevConv {
 public:
  explicit DevConv(const ConvLayer& L) : w_(L.weight) {
    if (!L.bias.empty()) b_ = std::make_unique<DevBuf<float>>(L.bias);
    d_ = {L.c_in, L.c_out, L.k, L.stride, w_.get(), b_ ? b_->get() : nullptr};
  }
  const sige_conv_desc* get() const { return &d_; }

 private:
  DevBuf<float> w_;
  std::unique_ptr<DevBuf<float>> b_;
  sige_conv_desc d_{};
};

inline Tensor download_tensor(const DevBuf<float>& d, int n, int c, int h, int w) {
  Tensor t(n, c, h, w);
  d.download(t.data.data(), t.data.size());
  return t;
}

// ---- mask reduction (mask.hpp) ----------------------------------------------

inline DifferenceMask compute_difference_mask(const Tensor& original, const Tensor& edited, float threshold) {
  require_same_shape(original, edited, "compute_difference_mask");
  DevBuf<float> o(original.data), e(edited.data);
  DevBuf<uint8_t> m(static_cast<size_t>(original.h) * original.w);
  check(sige_compute_difference_mask(o.get(), e.get(), original.n, original.c, original.h, original.w, threshold,
                                     m.get(), nullptr));
  DifferenceMask out(original.h, original.w);
  m.download(out.bits.data(), out.bits.size());
  return out;
}

inline DifferenceMask downsample_mask(const DifferenceMask& mask, int out_h, int out_w) {
  DevBuf<uint8_t> m(mask.bits), o(static_cast<size_t>(std::max(out_h, 0)) * std::max(out_w, 0));
  check(sige_downsample_mask(m.get(), mask.h, mask.w, out_h, out_w, o.get(), nullptr));
  DifferenceMask out(out_h, out_w);
  o.download(out.bits.data(), out.bits.size());
  return out;
}

inline DifferenceMask dilate_mask(const DifferenceMask& mask, int radius) {
  DevBuf<uint8_t> m(mask.bits), o(mask.bits.size());
  check(sige_dilate_mask(m.get(), mask.h, mask.w, radius, o.get(), nullptr));
  DifferenceMask out(mask.h, mask.w);
  o.download(out.bits.data(), out.bits.size());
  return out;
}

inline BlockIndexSet mask_to_block_indices(const DifferenceMask& mask, int block_size, int batch) {
  const int b = std::max(block_size, 1);
  const int cap = ((mask.h + b - 1) / b) * ((mask.w + b - 1) / b) * std::max(batch, 1);
  DevBuf<uint8_t> m(mask.bits);
  DevBuf<int32_t> idx(static_cast<size_t>(std::max(cap, 1)) * 3);
  int count = 0;
  check(sige_mask_to_block_indices(m.get(), mask.h, mask.w, block_size, batch, idx.get(), cap, &count, nullptr));
  std::vector<int32_t> host(static_cast<size_t>(count) * 3);
  idx.download(host.data(), host.size());
  return download_indices(host.data(), count, block_size, mask.h, mask.w);
}

// ---- block kernels (kernels.hpp) --------------------------------------------

inline BlockStack gather(const Tensor& x, const BlockIndexSet& idx, int k, int stride, const Epilogue& epilogue = {}) {
  DevBuf<float> xd(x.data);
  DevBuf<int32_t> id = upload_indices(idx);
  DevEpilogue e(epilogue);
  const int win = stride * idx.block_size + k - stride;
  BlockStack out;
  out.channels = x.c;
  out.block = idx.block_size;
  out.overlap = win - idx.block_size;
  out.origin = idx;
  out.data.resize(idx.count() * static_cast<size_t>(x.c) * std::max(win, 0) * std::max(win, 0));
  DevBuf<float> od(out.data.size());
  check(sige_gather(xd.get(), x.n, x.c, x.h, x.w, id.get(), static_cast<int>(idx.count()), idx.block_size, idx.h,
                    idx.w, k, stride, e.get(), od.get(), nullptr));
  od.download(out.data.data(), out.data.size());
  return out;
}

inline void scatter_inplace(const BlockStack& blocks, Tensor& base) {
  DevBuf<float> bd(blocks.data), td(base.data);
  DevBuf<int32_t> id = upload_indices(blocks.origin);
  check(sige_scatter_inplace(bd.get(), static_cast<int>(blocks.count()), blocks.channels, blocks.block, id.get(),
                             td.get(), base.n, base.c, base.h, base.w, nullptr));
  td.download(base.data.data(), base.data.size());
}

inline Tensor scatter(const BlockStack& blocks, const Tensor& base) {
  Tensor out = base;
  b200::scatter_inplace(blocks, out);
  return out;
}

inline void scatter_add_inplace(const BlockStack& blocks, Tensor& base) {
  DevBuf<float> bd(blocks.data), td(base.data);
  DevBuf<int32_t> id = upload_indices(blocks.origin);
  check(sige_scatter_add_inplace(bd.get(), static_cast<int>(blocks.count()), blocks.channels, blocks.block, id.get(),
                                 td.get(), base.n, base.c, base.h, base.w, nullptr));
  td.download(base.data.data(), base.data.size());
}

inline ScatterMap build_scatter_map(const BlockIndexSet& producer_idx) {
  static_assert(sizeof(ScatterMap::Entry) == sizeof(sige_scatter_entry), "ScatterMap::Entry layout");
  DevBuf<int32_t> id = upload_indices(producer_idx);
  DevBuf<sige_scatter_entry> md(static_cast<size_t>(producer_idx.h) * producer_idx.w);
  int bps = 0;
  check(sige_build_scatter_map(id.get(), static_cast<int>(producer_idx.count()), producer_idx.block_size,
                               producer_idx.h, producer_idx.w, md.get(), &bps, nullptr));
  ScatterMap m;
  m.h = producer_idx.h;
  m.w = producer_idx.w;
  m.block_size = producer_idx.block_size;
  m.blocks_per_sample = bps;
  m.cells.resize(md.size());
  std::vector<sige_scatter_entry> host = md.to_host();
  std::memcpy(m.cells.data(), host.data(), host.size() * sizeof(sige_scatter_entry));
  return m;
}

inline BlockStack scatter_gather(const BlockStack& blocks, const Tensor& original_out, const ScatterMap& map,
                                 const BlockIndexSet& consumer_idx, int k, int stride, const Epilogue& epilogue) {
  DevBuf<float> bd(blocks.data), od(original_out.data);
  DevBuf<sige_scatter_entry> md(map.cells.size());
  md.upload(reinterpret_cast<const sige_scatter_entry*>(map.cells.data()), map.cells.size());
  DevBuf<int32_t> ci = upload_indices(consumer_idx);
  DevEpilogue e(epilogue);
  const int win = stride * consumer_idx.block_size + k - stride;
  BlockStack out;
  out.channels = original_out.c;
  out.block = consumer_idx.block_size;
  out.overlap = win - consumer_idx.block_size;
  out.origin = consumer_idx;
  out.data.resize(consumer_idx.count() * static_cast<size_t>(original_out.c) * win * win);
  DevBuf<float> res(out.data.size());
  check(sige_scatter_gather(bd.get(), static_cast<int>(blocks.count()), blocks.block, od.get(), original_out.n,
                            original_out.c, original_out.h, original_out.w, md.get(), map.blocks_per_sample, ci.get(),
                            static_cast<int>(consumer_idx.count()), consumer_idx.block_size, consumer_idx.h,
                            consumer_idx.w, k, stride, e.get(), res.get(), nullptr));
  res.download(out.data.data(), out.data.size());
  return out;
}

namespace detail {
using ResidualFn = int (*)(const float*, int, int, const int32_t*, const float*, int, int, const int32_t*, const float*,
                           const float*, float*, int, int, int, int, sige_stream_t);
inline Tensor residual(ResidualFn fn, const BlockStack& m, const BlockStack& s, const Tensor& sum, const Tensor& osc) {
  DevBuf<float> md(m.data), sd(s.data), sumd(sum.data), oscd(osc.data), out(sum.data.size());
  DevBuf<int32_t> mi = upload_indices(m.origin), si = upload_indices(s.origin);
  check(fn(md.get(), static_cast<int>(m.count()), m.block, mi.get(), sd.get(), static_cast<int>(s.count()), s.block,
           si.get(), sumd.get(), oscd.get(), out.get(), sum.n, sum.c, sum.h, sum.w, nullptr));
  return download_tensor(out, sum.n, sum.c, sum.h, sum.w);
}
inline BlockStack combine(const BlockStack& a, const BlockStack& b, float sign) {
  if (a.channels != b.channels || a.block != b.block || a.overlap != b.overlap || a.count() != b.count())
    throw ConfigError(sign > 0 ? "add_blocks: block stack geometry mismatch" : "subtract_blocks: block stack geometry mismatch");
  DevBuf<float> ad(a.data), bd(b.data), od(a.data.size());
  check(sige_combine_blocks(ad.get(), bd.get(), sign, a.data.size(), od.get(), nullptr));
  BlockStack out = a;
  od.download(out.data.data(), out.data.size());
  return out;
}
}  // namespace detail

inline Tensor scatter_with_block_residual(const BlockStack& main_blocks, const BlockStack& shortcut_blocks,
                                          const Tensor& precomputed_sum, const Tensor& original_shortcut) {
  return detail::residual(sige_scatter_with_block_residual, main_blocks, shortcut_blocks, precomputed_sum,
                          original_shortcut);
}

inline Tensor scatter_with_block_residual_unfused(const BlockStack& main_blocks, const BlockStack& shortcut_blocks,
                                                  const Tensor& precomputed_sum, const Tensor& original_shortcut) {
  return detail::residual(sige_scatter_with_block_residual_unfused, main_blocks, shortcut_blocks, precomputed_sum,
                          original_shortcut);
}

inline BlockStack add_blocks(const BlockStack& a, const BlockStack& b) { return detail::combine(a, b, 1.0f); }
inline BlockStack subtract_blocks(const BlockStack& a, const BlockStack& b) { return detail::combine(a, b, -1.0f); }

inline void apply_epilogue_on_blocks(BlockStack& blocks, const Epilogue& epilogue) {
  DevBuf<float> bd(blocks.data);
  DevBuf<int32_t> id = upload_indices(blocks.origin);
  DevEpilogue e(epilogue);
  check(sige_apply_epilogue_on_blocks(bd.get(), static_cast<int>(blocks.count()), blocks.channels, blocks.bh(),
                                      id.get(), e.get(), nullptr));
  bd.download(blocks.data.data(), blocks.data.size());
}

// math: SIGE_MATH_EXACT (the reference's arithmetic, bit-exact), _FP32_FMA,
// _TF32 or _F16 (tcgen05 tensor cores).
inline BlockStack conv_on_blocks(const BlockStack& blocks, const ConvLayer& layer, bool with_bias = true,
                                 int math = SIGE_MATH_EXACT) {
  DevBuf<float> bd(blocks.data);
  DevConv cv(layer);
  const int b = blocks.bh() >= layer.k ? (blocks.bh() - layer.k) / layer.stride + 1 : 0;
  BlockStack out;
  out.channels = layer.c_out;
  out.block = b;
  out.overlap = 0;
  out.origin = blocks.origin;
  out.data.resize(blocks.count() * static_cast<size_t>(layer.c_out) * b * b);
  DevBuf<float> od(out.data.size());
  check(sige_conv_on_blocks(bd.get(), static_cast<int>(blocks.count()), blocks.bh(), cv.get(), with_bias ? 1 : 0, math,
                            od.get(), blocks.block, nullptr));
  od.download(out.data.data(), out.data.size());
  return out;
}

inline Tensor conv2d(const Tensor& input, const ConvLayer& layer, bool with_bias = true, int math = SIGE_MATH_EXACT) {
  DevBuf<float> xd(input.data);
  DevConv cv(layer);
  const int oh = conv_out_dim(input.h, layer.k, layer.stride), ow = conv_out_dim(input.w, layer.k, layer.stride);
  DevBuf<float> od(static_cast<size_t>(input.n) * layer.c_out * oh * ow);
  check(sige_conv2d(xd.get(), input.n, input.c, input.h, input.w, cv.get(), with_bias ? 1 : 0, math, od.get(), nullptr));
  return download_tensor(od, input.n, layer.c_out, oh, ow);
}

// ---- models, RunConfig, the executor (graph.hpp) ----------------------------

// sige::ModelSpec (graph.hpp:63-71) -> sige_model_desc; weights borrowed from `m`.
class ModelView {
 public:
  explicit ModelView(const ModelSpec& m) : name_(m.name) {
    auto conv = [](const ConvLayer& c) {
      return sige_conv_desc{c.c_in, c.c_out, c.k, c.stride, c.weight.data(), c.bias.empty() ? nullptr : c.bias.data()};
    };
    auto norm = [](const NormLayer& n) {
      return sige_norm_desc{static_cast<int>(n.kind), n.groups, n.channels(), n.eps, n.gamma.data(), n.beta.data(),
                            n.running_mean.empty() ? nullptr : n.running_mean.data(),
                            n.running_var.empty() ? nullptr : n.running_var.data()};
    };
    for (const Layer& L : m.layers) {
      sige_layer_desc d{};
      d.kind = static_cast<int>(L.kind);
      d.policy_sparse = L.policy.sparse ? 1 : 0;
      d.min_resolution = L.policy.min_resolution;
      if (L.kind == LayerKind::Conv || L.kind == LayerKind::Downsample) d.conv = conv(L.conv);
      if (L.kind == LayerKind::Norm) d.norm = norm(L.norm);
      if (L.kind == LayerKind::Activation) d.act = static_cast<int>(L.act);
      if (L.kind == LayerKind::ResBlock) {
        d.conv = conv(L.res.conv1);
        d.conv2 = conv(L.res.conv2);
        d.norm = norm(L.res.norm);
        d.act = static_cast<int>(L.res.act);
        d.has_shortcut = L.res.shortcut.has_value() ? 1 : 0;
        if (d.has_shortcut) d.shortcut = conv(*L.res.shortcut);
      }
      layers_.push_back(d);
    }
    desc_ = {name_.c_str(), m.in_channels, m.in_h, m.in_w, static_cast<int>(layers_.size()), layers_.data()};
  }
  const sige_model_desc* get() const { return &desc_; }
  uint64_t weight_hash() const { return sige_model_weight_hash(&desc_); }  // models.cpp:185-207

 private:
  std::string name_;
  std::vector<sige_layer_desc> layers_;
  sige_model_desc desc_{};
};

inline sige_run_config to_c(const RunConfig& c) {
  return {c.step, c.mask_threshold, c.dilate_full, c.dilate_scale, c.block3, c.block1, c.min_sparse_res,
          c.sparse ? 1 : 0, c.norm_precompute ? 1 : 0, c.elem_fusion ? 1 : 0, c.scatter_fusion ? 1 : 0, c.seed};
}

// precompute + sparse_forward (graph.hpp:168-226) on one B200: the model and
// its ActivationCache stay resident in HBM inside the engine.
class Engine {
 public:
  Engine(const ModelSpec& m, int batch, int math = SIGE_MATH_F16) : view_(m), batch_(batch) {
    check(sige_engine_create(view_.get(), batch, math, &e_));
  }
  ~Engine() { sige_engine_destroy(e_); }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  void precompute(const Tensor& original, int step = 0) {  // the dense walk runs on the device
    DevBuf<float> d(original.data);
    check(sige_engine_precompute(e_, d.get(), step, nullptr));
    cuda_check(cudaDeviceSynchronize(), "precompute");
  }
  Tensor sparse_forward(const Tensor& edited, const DifferenceMask& mask, const RunConfig& cfg) {
    int n, c, h, w;
    check(sige_engine_output_shape(e_, &n, &c, &h, &w));
    if (mask.h != edited.h || mask.w != edited.w)  // check_inputs (graph.cpp:606-614)
      throw ConfigError("forward: mask is " + std::to_string(mask.h) + "x" + std::to_string(mask.w) + " but input is " +
                        std::to_string(edited.h) + "x" + std::to_string(edited.w));
    Tensor out(n, c, h, w);
    const sige_run_config rc = to_c(cfg);
    check(sige_engine_sparse_forward_host(e_, edited.data.data(), mask.bits.data(), &rc, out.data.data(), nullptr));
    return out;
  }
  Tensor dense_forward(const Tensor& input) {
    int n, c, h, w;
    check(sige_engine_output_shape(e_, &n, &c, &h, &w));
    DevBuf<float> in(input.data), out(static_cast<size_t>(n) * c * h * w);
    check(sige_engine_dense_forward(e_, in.get(), 0, 0, out.get(), nullptr));
    return download_tensor(out, n, c, h, w);
  }
  Tensor cached(const std::string& key, int n, int c, int h, int w, int step = 0) {  // ActivationCache::tensor_entry
    Tensor t(n, c, h, w);
    check(sige_engine_get_tensor(e_, step, key.c_str(), t.data.data(), t.data.size()));
    return t;
  }
  // RunTrace rows of the last call (graph.hpp:194-216): {blocks, gathered,
  // scattered, macs, dense_macs, ran_sparse}; empty after the empty-mask
  // short-circuit (graph.cpp:665-668).
  std::vector<std::array<uint64_t, 6>> trace() {
    std::vector<uint64_t> rows(6 * 1024);
    int nrows = 0;
    check(sige_engine_trace(e_, rows.data(), 1024, &nrows, nullptr));
    std::vector<std::array<uint64_t, 6>> out(nrows);
    for (int i = 0; i < nrows; ++i)
      for (int j = 0; j < 6; ++j) out[i][j] = rows[6 * i + j];
    return out;
  }

 private:
  ModelView view_;
  int batch_;
  sige_engine* e_ = nullptr;
};

}  // namespace b200
}  // namespace sige
