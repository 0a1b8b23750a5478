// The reference's own acceptance criteria 1, 3 and 5
// (proj/tests/acceptance.cpp:52-253, 306-330) run through the C++ adapter
// include/sige_b200.hpp, i.e. through libsige_b200's C ABI on the GPU, with
// the unmodified reference (compiled with -Dsige=sigeref) as the checker.
//
//   adapter_acceptance cpu   host-only checks of the adapter (no device):
//                            ModelView reproduces model_weight_hash of every
//                            toy model, RunConfig conversion, ConfigError
//                            mapping of a library-side validation failure
//   adapter_acceptance gpu   criteria 1, 3, 5 (one [PASS]/[FAIL] line each)
//
// Exit 0 iff every executed check passed.
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sige/fixtures.hpp"
#include "sige/models.hpp"
#include "sige_b200.hpp"

using namespace sige;

namespace {

int g_failed = 0;

void report(const char* name, bool ok, const std::string& detail) {
  std::printf("[%s] %s: %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
  if (!ok) ++g_failed;
}

bool same_bits(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
}

ConvLayer rand_conv(Rng& rng, int c_in, int c_out, int k, int stride) {  // acceptance.cpp:38-51
  ConvLayer L;
  L.c_in = c_in;
  L.c_out = c_out;
  L.k = k;
  L.stride = stride;
  const float bound = 1.0f / std::sqrt(static_cast<float>(c_in) * k * k);
  L.weight.resize(static_cast<size_t>(c_out) * c_in * k * k);
  for (float& v : L.weight) v = rng.uniform(-bound, bound);
  L.bias.resize(c_out);
  for (float& v : L.bias) v = rng.uniform(-0.1f, 0.1f);
  return L;
}

// ---- host-only ----------------------------------------------------------
void cpu_checks() {
  bool ok = true;
  std::string bad;
  for (const std::string& name : toy_model_names()) {
    const ModelSpec m = toy_model(name);
    const b200::ModelView v(m);
    if (v.weight_hash() != model_weight_hash(m)) {
      ok = false;
      bad += name + " ";
    }
  }
  report("model-view", ok, ok ? "ModelView reproduces model_weight_hash of every toy model" : "hash differs: " + bad);

  RunConfig c;
  c.dilate_full = 5;
  c.min_sparse_res = 64;
  c.elem_fusion = false;
  const sige_run_config rc = b200::to_c(c);
  report("run-config", rc.dilate_full == 5 && rc.min_sparse_res == 64 && rc.elem_fusion == 0 && rc.block3 == 6 &&
                           rc.block1 == 4 && rc.sparse == 1 && std::fabs(rc.mask_threshold - 1e-3f) == 0.0f,
         "RunConfig -> sige_run_config field by field");

  // A model whose channels do not chain: the library rejects it (before any
  // device work) with a ConfigError that surfaces as sige::ConfigError.
  ModelSpec bad_m = toy_model("conv3x3_128");
  bad_m.in_channels += 1;
  try {
    b200::Engine e(bad_m, 1, SIGE_MATH_EXACT);
    report("config-error", false, "no error raised");
  } catch (const ConfigError& e) {
    report("config-error", std::strlen(e.what()) > 0, std::string("sige::ConfigError: ") + e.what());
  }
}

// ---- criterion 1: random single-conv sparse updates (acceptance.cpp:52-170)
struct ConvCase {
  ModelSpec model;
  Tensor original, edited;
  DifferenceMask mask;
  RunConfig config;
};

ConvCase conv_case(Rng& rng) {  // make_conv_case: same draws, same order
  ConvCase cs;
  const int res = 2 * rng.uniform_int(8, 32);
  const int c_in = rng.uniform_int(4, 32), c_out = rng.uniform_int(4, 32);
  const int k = rng.uniform_int(0, 1) == 0 ? 1 : 3;
  const int stride = rng.uniform_int(1, 2);
  const int batch = rng.uniform_int(0, 9) == 0 ? 2 : 1;
  cs.model.name = "case_conv";
  cs.model.in_channels = c_in;
  cs.model.in_h = cs.model.in_w = res;
  Layer L;
  L.kind = LayerKind::Conv;
  L.name = "conv";
  L.conv = rand_conv(rng, c_in, c_out, k, stride);
  cs.model.layers = {L};
  cs.original = Tensor(batch, c_in, res, res);
  fill_uniform(cs.original, rng, -1.0f, 1.0f);
  cs.edited = cs.original;
  const float frac = rng.uniform(0.01f, 0.40f);
  const int side = std::max(1, static_cast<int>(std::lround(res * std::sqrt(frac))));
  const int r0 = rng.uniform_int(0, res - side), c0 = rng.uniform_int(0, res - side);
  for (int n = 0; n < batch; ++n)
    for (int c = 0; c < c_in; ++c)
      for (int y = r0; y < r0 + side; ++y)
        for (int x = c0; x < c0 + side; ++x) {
          const float mag = rng.uniform(0.1f, 0.6f);
          cs.edited.at(n, c, y, x) += rng.uniform(0.0f, 1.0f) < 0.5f ? -mag : mag;
        }
  cs.mask = compute_difference_mask(cs.original, cs.edited, 1e-3f);
  cs.config.dilate_full = rng.uniform_int(1, 3);
  cs.config.seed = rng.next_u32();
  return cs;
}

void criterion_1() {
  Rng rng(9001);
  float worst = 0.0f;
  int ref_bit_exact = 0;
  for (int i = 0; i < 200; ++i) {
    ConvCase cs = conv_case(rng);
    ActivationCache cache;
    precompute(cache, cs.model, cs.original);  // the reference cache (checker only)
    b200::Engine eng(cs.model, cs.original.n, SIGE_MATH_EXACT);
    eng.precompute(cs.original);
    const Tensor sparse = eng.sparse_forward(cs.edited, cs.mask, cs.config);
    const Tensor dense = dense_forward(cs.model, cs.edited);
    const Tensor& cached = cache.final_output(0);
    const DifferenceMask cov = output_coverage(cs.model, cs.mask, cs.edited.n, cs.config);
    for (int n = 0; n < sparse.n; ++n)
      for (int c = 0; c < sparse.c; ++c)
        for (int y = 0; y < sparse.h; ++y)
          for (int x = 0; x < sparse.w; ++x) {
            const float s = sparse.at(n, c, y, x);
            if (cov.at(y, x)) {
              const float d = std::fabs(s - dense.at(n, c, y, x));
              worst = std::max(worst, d);
              if (d > 1e-5f) {
                report("criterion-1", false, "case " + std::to_string(i) + ": covered diff " + std::to_string(d));
                return;
              }
            } else if (s != cached.at(n, c, y, x)) {
              report("criterion-1", false, "case " + std::to_string(i) + ": uncovered pixel differs from cache");
              return;
            }
          }
    ref_bit_exact += same_bits(sparse.data, sparse_forward(cs.model, cs.edited, cache, cs.mask, cs.config).data);
  }
  char buf[200];
  std::snprintf(buf, sizeof buf,
                "200 cases through b200::Engine: worst covered diff vs dense %.2e (tol 1e-5), uncovered bit-exact, "
                "%d/200 bit-identical to sigeref::sparse_forward",
                worst, ref_bit_exact);
  report("criterion-1", ref_bit_exact == 200, buf);
}

// ---- criterion 3: fused scatter-gather / residual join (acceptance.cpp:172-253)
void criterion_3() {
  Rng rng(9002);
  int same_as_ref = 0;
  for (int i = 0; i < 200; ++i) {
    const int res = 2 * rng.uniform_int(8, 16);
    const int c_in = rng.uniform_int(4, 16), c_out = rng.uniform_int(4, 16);
    const int batch = rng.uniform_int(0, 4) == 0 ? 2 : 1;
    const ConvLayer conv1 = rand_conv(rng, c_in, c_out, 3, 1);
    const ConvLayer conv2 = rand_conv(rng, c_out, c_out, 3, 1);
    const ConvLayer proj = rand_conv(rng, c_in, c_out, 1, 1);
    Tensor orig(batch, c_in, res, res);
    fill_uniform(orig, rng, -1.0f, 1.0f);
    Tensor edit = orig;
    for (int rep = 0; rep < 4; ++rep)
      for (int n = 0; n < batch; ++n)
        for (int c = 0; c < c_in; ++c) {
          const int y = rng.uniform_int(0, res - 1);
          const int x = rng.uniform_int(0, res - 1);
          edit.at(n, c, y, x) += 0.7f;
        }
    // mask reduction through the adapter, cross-checked against the reference
    const DifferenceMask mask = b200::compute_difference_mask(orig, edit, 1e-3f);
    const DifferenceMask dil = b200::dilate_mask(mask, rng.uniform_int(1, 2));
    const BlockIndexSet idx_m = b200::mask_to_block_indices(dil, 6, batch);
    const BlockIndexSet idx_s = b200::mask_to_block_indices(dil, 4, batch);
    bool ok = mask.bits == compute_difference_mask(orig, edit, 1e-3f).bits &&
              idx_m.content_hash() == mask_to_block_indices(dil, 6, batch).content_hash() &&
              idx_s.content_hash() == mask_to_block_indices(dil, 4, batch).content_hash();
    Epilogue epi;
    if (i % 2 == 0) {
      std::vector<float> scale(c_out), shift(c_out);
      for (int c = 0; c < c_out; ++c) {
        scale[c] = rng.uniform(0.5f, 1.5f);
        shift[c] = rng.uniform(-0.3f, 0.3f);
      }
      epi.add_scale_shift(std::move(scale), std::move(shift));
      epi.add_activation(ActKind::Silu);
    }
    // scatter-gather: fused vs materialise-then-gather, bit-exact
    const BlockStack m1 = b200::conv_on_blocks(b200::gather(edit, idx_m, 3, 1), conv1);
    const Tensor base1 = b200::conv2d(orig, conv1);
    const ScatterMap map1 = b200::build_scatter_map(idx_m);
    const BlockStack fused_sg = b200::scatter_gather(m1, base1, map1, idx_m, 3, 1, epi);
    Tensor full1 = b200::scatter(m1, base1);
    epi.apply_tensor(full1);
    const BlockStack staged_sg = b200::gather(full1, idx_m, 3, 1);
    if (fused_sg.data != staged_sg.data) {
      report("criterion-3", false, "case " + std::to_string(i) + ": scatter-gather not bit-exact");
      return;
    }
    // residual join: fused vs the unfused kernel twin, bit-exact
    const BlockStack m2 = b200::conv_on_blocks(staged_sg, conv2);
    const BlockStack scb = b200::conv_on_blocks(b200::gather(edit, idx_s, 1, 1), proj);
    Tensor orig_mid = b200::conv2d(orig, conv1);
    epi.apply_tensor(orig_mid);
    const Tensor orig_sc = b200::conv2d(orig, proj);
    const Tensor sum = add(b200::conv2d(orig_mid, conv2), orig_sc);
    const Tensor fused = b200::scatter_with_block_residual(m2, scb, sum, orig_sc);
    const Tensor staged = b200::scatter_with_block_residual_unfused(m2, scb, sum, orig_sc);
    if (!same_bits(fused.data, staged.data)) {
      report("criterion-3", false, "case " + std::to_string(i) + ": residual join not bit-exact");
      return;
    }
    // and every adapter result equals the reference's own
    const BlockStack r_m1 = conv_on_blocks(gather(edit, idx_m, 3, 1), conv1);
    const BlockStack r_sg = scatter_gather(r_m1, conv2d(orig, conv1), build_scatter_map(idx_m), idx_m, 3, 1, epi);
    const BlockStack r_m2 = conv_on_blocks(r_sg, conv2);
    const BlockStack r_scb = conv_on_blocks(gather(edit, idx_s, 1, 1), proj);
    ok = ok && same_bits(m1.data, r_m1.data) && same_bits(fused_sg.data, r_sg.data) &&
         same_bits(fused.data, scatter_with_block_residual(r_m2, r_scb, sum, orig_sc).data) &&
         same_bits(scb.data, r_scb.data);
    same_as_ref += ok;
  }
  char buf[200];
  std::snprintf(buf, sizeof buf,
                "200 cases: fused == unfused bit-exact for scatter-gather and residual join; %d/200 cases "
                "bit-identical to the reference's own results",
                same_as_ref);
  report("criterion-3", same_as_ref == 200, buf);
}

// ---- criterion 5: empty mask short-circuit (acceptance.cpp:306-330)
void criterion_5() {
  const ModelSpec m = toy_model("mini_unet_gn");
  const EditFixture fx = make_edit_fixture("rect5", 1, 3, 64, 64, 7);
  b200::Engine eng(m, 1, SIGE_MATH_F16);
  eng.precompute(fx.original);
  const DifferenceMask empty(64, 64);
  RunConfig cfg;
  cfg.norm_precompute = true;
  const Tensor out = eng.sparse_forward(fx.original, empty, cfg);
  const Tensor cached = eng.cached("final", out.n, out.c, out.h, out.w);
  const auto tr = eng.trace();
  const bool ok = same_bits(out.data, cached.data) && tr.empty();
  report("criterion-5", ok,
         std::string("empty mask: output ") + (same_bits(out.data, cached.data) ? "bit-identical" : "DIFFERS") +
             " to the cached final output, " + std::to_string(tr.size()) + " trace rows (short-circuit)");
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  try {
    if (mode == "cpu") {
      cpu_checks();
    } else {
      criterion_1();
      criterion_3();
      criterion_5();
    }
  } catch (const std::exception& e) {
    report("exception", false, e.what());
  }
  return g_failed == 0 ? 0 : 1;
}
