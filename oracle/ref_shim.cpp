// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// An extern "C" veneer over the UNMODIFIED reference library, compiled from
// /root/reference/proj/src with -Dsige=sigeref by oracle/Makefile into
// oracle/_ref/libsigeref.so. It lets the Python tests (and bench.py's
// cpu_baseline / --impl reference leg) drive the reference's own public API:
// proj/include/sige/{mask,kernels,conv,norm,eltwise,graph,fixtures,models}.hpp.
// No reference source is copied; this file only calls it.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "sige/common.hpp"
#include "sige/conv.hpp"
#include "sige/eltwise.hpp"
#include "sige/fixtures.hpp"
#include "sige/graph.hpp"
#include "sige/kernels.hpp"
#include "sige/mask.hpp"
#include "sige/models.hpp"
#include "sige/norm.hpp"
#include "sige/tensor.hpp"
#ifdef SIGE_REF_IO
#include "sige/io.hpp"
#endif
#include "sige_b200.h"

using namespace sigeref;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return SIGE_ERR_CONFIG;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SIGE_ERR_INTERNAL;
  }
}

Tensor to_tensor(const float* p, int n, int c, int h, int w) {
  Tensor t(n, c, h, w);
  std::memcpy(t.data.data(), p, t.data.size() * sizeof(float));
  return t;
}

void from_tensor(const Tensor& t, float* out) {
  std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
}

DifferenceMask to_mask(const uint8_t* m, int h, int w) {
  DifferenceMask d(h, w);
  std::memcpy(d.bits.data(), m, static_cast<size_t>(h) * w);
  return d;
}

BlockIndexSet to_index_set(const int32_t* idx, int count, int block, int h, int w) {
  BlockIndexSet s;
  s.block_size = block;
  s.h = h;
  s.w = w;
  s.indices.resize(count);
  for (int i = 0; i < count; ++i) s.indices[i] = {idx[3 * i], idx[3 * i + 1], idx[3 * i + 2]};
  return s;
}

BlockStack to_stack(const float* p, int count, int channels, int block, int overlap,
                    const BlockIndexSet& origin) {
  BlockStack b;
  b.channels = channels;
  b.block = block;
  b.overlap = overlap;
  b.origin = origin;
  b.data.assign(p, p + static_cast<size_t>(count) * b.block_stride());
  return b;
}

Epilogue to_epilogue(const sige_epilogue* e) {
  Epilogue out;
  if (!e) return out;
  for (int i = 0; i < e->num_steps; ++i) {
    const sige_epilogue_step& s = e->steps[i];
    if (s.kind == SIGE_EPI_SCALE_SHIFT) {
      out.add_scale_shift(std::vector<float>(s.scale, s.scale + s.nparams),
                          std::vector<float>(s.shift, s.shift + s.nparams));
    } else {
      out.add_activation(static_cast<ActKind>(s.act));
    }
  }
  return out;
}

ConvLayer to_conv(const sige_conv_desc& d) {
  ConvLayer c;
  c.c_in = d.c_in;
  c.c_out = d.c_out;
  c.k = d.k;
  c.stride = d.stride;
  c.weight.assign(d.weight, d.weight + static_cast<size_t>(d.c_out) * d.c_in * d.k * d.k);
  if (d.bias) c.bias.assign(d.bias, d.bias + d.c_out);
  return c;
}

NormLayer to_norm(const sige_norm_desc& d) {
  NormLayer n;
  n.kind = static_cast<NormKind>(d.kind);
  n.groups = d.groups;
  n.eps = d.eps;
  n.gamma.assign(d.gamma, d.gamma + d.channels);
  n.beta.assign(d.beta, d.beta + d.channels);
  if (d.running_mean) n.running_mean.assign(d.running_mean, d.running_mean + d.channels);
  if (d.running_var) n.running_var.assign(d.running_var, d.running_var + d.channels);
  return n;
}

RunConfig to_config(const sige_run_config* c) {
  RunConfig r;
  if (!c) return r;
  r.step = c->step;
  r.mask_threshold = c->mask_threshold;
  r.dilate_full = c->dilate_full;
  r.dilate_scale = c->dilate_scale;
  r.block3 = c->block3;
  r.block1 = c->block1;
  r.min_sparse_res = c->min_sparse_res;
  r.sparse = c->sparse != 0;
  r.norm_precompute = c->norm_precompute != 0;
  r.elem_fusion = c->elem_fusion != 0;
  r.scatter_fusion = c->scatter_fusion != 0;
  r.seed = c->seed;
  return r;
}

// Config 1 and config 2 of BASELINE.json, built with the reference's own
// types and Rng, following the recipe DESIGN.md §"Synthetic workloads" fixes
// (models.cpp:91-100 style). The product library and the C restatement build
// the same models; tests compare model_weight_hash across all three.
ConvLayer make_conv(Rng& rng, int c_in, int c_out, int k, int stride) {
  ConvLayer c;
  c.c_in = c_in;
  c.c_out = c_out;
  c.k = k;
  c.stride = stride;
  float bound = 1.0f / std::sqrt(static_cast<float>(c_in * k * k));
  c.weight.resize(static_cast<size_t>(c_out) * c_in * k * k);
  for (float& v : c.weight) v = rng.uniform(-bound, bound);
  c.bias.resize(c_out);
  for (float& v : c.bias) v = rng.uniform(-0.05f, 0.05f);
  return c;
}

NormLayer make_gn(Rng& rng, int channels, int groups) {
  NormLayer n;
  n.kind = NormKind::Group;
  n.groups = groups;
  n.gamma.resize(channels);
  n.beta.resize(channels);
  for (float& v : n.gamma) v = rng.uniform(0.8f, 1.2f);
  for (float& v : n.beta) v = rng.uniform(-0.1f, 0.1f);
  return n;
}

Layer conv_l(Rng& rng, const std::string& name, int ci, int co, int k, int s) {
  Layer L;
  L.kind = s == 2 ? LayerKind::Downsample : LayerKind::Conv;
  L.name = name;
  L.conv = make_conv(rng, ci, co, k, s);
  return L;
}

Layer rb_l(Rng& rng, const std::string& name, int ci, int co) {
  Layer L;
  L.kind = LayerKind::ResBlock;
  L.name = name;
  L.res.conv1 = make_conv(rng, ci, co, 3, 1);
  L.res.norm = make_gn(rng, co, 32);
  L.res.act = ActKind::Silu;
  L.res.conv2 = make_conv(rng, co, co, 3, 1);
  if (ci != co) L.res.shortcut = make_conv(rng, ci, co, 1, 1);
  return L;
}

ModelSpec build_single_conv64() {
  Rng rng(1001);
  ModelSpec m;
  m.name = "single_conv64";
  m.in_channels = 64;
  m.in_h = 256;
  m.in_w = 256;
  m.layers.push_back(conv_l(rng, "conv", 64, 64, 3, 1));
  return m;
}

ModelSpec build_ddim_stack(int res, int base) {
  Rng rng(2211);
  ModelSpec m;
  m.name = "ddim_stack";
  m.in_channels = 3;
  m.in_h = res;
  m.in_w = res;
  const int mult[6] = {1, 1, 2, 2, 4, 4};
  m.layers.push_back(conv_l(rng, "conv_in", 3, base, 3, 1));
  int c = base;
  for (int lvl = 0; lvl < 6; ++lvl) {
    for (int j = 0; j < 2; ++j) {
      m.layers.push_back(rb_l(rng, "enc" + std::to_string(lvl) + "_rb" + std::to_string(j), c,
                              base * mult[lvl]));
      c = base * mult[lvl];
    }
    if (lvl < 5) m.layers.push_back(conv_l(rng, "down" + std::to_string(lvl), c, c, 3, 2));
  }
  for (int j = 0; j < 2; ++j) m.layers.push_back(rb_l(rng, "mid_rb" + std::to_string(j), c, c));
  for (int lvl = 0; lvl < 6; ++lvl) {
    int dc = base * mult[5 - lvl];
    for (int j = 0; j < 3; ++j) {
      m.layers.push_back(rb_l(rng, "dec" + std::to_string(lvl) + "_rb" + std::to_string(j), c, dc));
      c = dc;
    }
    if (lvl < 5) {
      Layer up;
      up.kind = LayerKind::Upsample;
      up.name = "up" + std::to_string(lvl);
      m.layers.push_back(up);
      m.layers.push_back(conv_l(rng, "upconv" + std::to_string(lvl), c, c, 3, 1));
    }
  }
  Layer norm;
  norm.kind = LayerKind::Norm;
  norm.name = "out_norm";
  norm.norm = make_gn(rng, c, 32);
  m.layers.push_back(norm);
  Layer act;
  act.kind = LayerKind::Activation;
  act.name = "out_act";
  act.act = ActKind::Silu;
  m.layers.push_back(act);
  m.layers.push_back(conv_l(rng, "conv_out", c, 3, 3, 1));
  return m;
}

ModelSpec build_named(const std::string& name) {
  if (name == "single_conv64") return build_single_conv64();
  if (name == "ddim_stack") return build_ddim_stack(256, 128);
  if (name == "ddim_stack_64x32") return build_ddim_stack(64, 32);
  return toy_model(name);
}

void write_trace(const RunTrace& tr, uint64_t* rows, int cap, int* nrows) {
  int n = 0;
  for (const TraceLayer& l : tr.layers) {
    if (n < cap && rows) {
      uint64_t* r = rows + 6 * n;
      r[0] = l.active_blocks;
      r[1] = l.gathered_elems;
      r[2] = l.scattered_elems;
      r[3] = l.macs;
      r[4] = l.dense_macs;
      r[5] = l.ran_sparse ? 1 : 0;
    }
    ++n;
  }
  if (nrows) *nrows = n;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

float ref_expf(float x) { return std::exp(x); }

// FNV-1a over expf output bits for every finite float in [lo, hi] taken in
// ascending bit order of the positive and negative ranges.
uint64_t ref_expf_digest(uint32_t bits_lo, uint32_t bits_hi) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t b = bits_lo; b <= bits_hi; ++b) {
    uint32_t u = static_cast<uint32_t>(b);
    float x;
    std::memcpy(&x, &u, 4);
    float y = std::exp(x);
    uint32_t o;
    std::memcpy(&o, &y, 4);
    h = fnv1a64(&o, 4, h);
  }
  return h;
}

uint64_t ref_fnv1a64(const void* p, size_t n, uint64_t seed) { return fnv1a64(p, n, seed); }

int ref_make_edit_fixture(const char* kind, int n, int c, int h, int w, uint32_t seed,
                          float* orig, float* edited) {
  return guarded([&] {
    EditFixture fx = make_edit_fixture(kind, n, c, h, w, seed);
    from_tensor(fx.original, orig);
    from_tensor(fx.edited, edited);
  });
}

int ref_rng_stream(uint32_t seed, int count, uint32_t* out_u32, float* out_uniform, float lo,
                   float hi) {
  Rng a(seed), b(seed);
  for (int i = 0; i < count; ++i) {
    if (out_u32) out_u32[i] = a.next_u32();
    if (out_uniform) out_uniform[i] = b.uniform(lo, hi);
  }
  return 0;
}

int ref_compute_difference_mask(const float* o, const float* e, int n, int c, int h, int w,
                                float thr, uint8_t* out) {
  return guarded([&] {
    DifferenceMask m = compute_difference_mask(to_tensor(o, n, c, h, w), to_tensor(e, n, c, h, w), thr);
    std::memcpy(out, m.bits.data(), m.bits.size());
  });
}

int ref_downsample_mask(const uint8_t* m, int h, int w, int oh, int ow, uint8_t* out) {
  return guarded([&] {
    DifferenceMask d = downsample_mask(to_mask(m, h, w), oh, ow);
    std::memcpy(out, d.bits.data(), d.bits.size());
  });
}

int ref_dilate_mask(const uint8_t* m, int h, int w, int r, uint8_t* out) {
  return guarded([&] {
    DifferenceMask d = dilate_mask(to_mask(m, h, w), r);
    std::memcpy(out, d.bits.data(), d.bits.size());
  });
}

int ref_mask_to_block_indices(const uint8_t* m, int h, int w, int b, int batch, int32_t* idx,
                              int cap, int* count, uint64_t* hash) {
  return guarded([&] {
    BlockIndexSet s = mask_to_block_indices(to_mask(m, h, w), b, batch);
    *count = static_cast<int>(s.count());
    if (hash) *hash = s.content_hash();
    for (int i = 0; i < *count && i < cap; ++i) {
      idx[3 * i] = s.indices[i].n;
      idx[3 * i + 1] = s.indices[i].r;
      idx[3 * i + 2] = s.indices[i].c;
    }
  });
}

int ref_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count, int b,
               int ih, int iw, int k, int s, const sige_epilogue* epi, float* out) {
  return guarded([&] {
    BlockStack g = gather(to_tensor(x, n, c, h, w), to_index_set(idx, count, b, ih, iw), k, s,
                          to_epilogue(epi));
    std::memcpy(out, g.data.data(), g.data.size() * sizeof(float));
  });
}

int ref_scatter(const float* blocks, int count, int channels, int block, const int32_t* idx,
                const float* base, float* out, int n, int c, int h, int w) {
  return guarded([&] {
    BlockStack bs = to_stack(blocks, count, channels, block, 0, to_index_set(idx, count, block, h, w));
    from_tensor(scatter(bs, to_tensor(base, n, c, h, w)), out);
  });
}

int ref_scatter_add_inplace(const float* blocks, int count, int channels, int block,
                            const int32_t* idx, float* base, int n, int c, int h, int w) {
  return guarded([&] {
    BlockStack bs = to_stack(blocks, count, channels, block, 0, to_index_set(idx, count, block, h, w));
    Tensor t = to_tensor(base, n, c, h, w);
    scatter_add_inplace(bs, t);
    from_tensor(t, base);
  });
}

int ref_build_scatter_map(const int32_t* idx, int count, int block, int h, int w,
                          sige_scatter_entry* out, int* bps) {
  return guarded([&] {
    ScatterMap m = build_scatter_map(to_index_set(idx, count, block, h, w));
    *bps = m.blocks_per_sample;
    for (size_t i = 0; i < m.cells.size(); ++i) {
      out[i].block = m.cells[i].block;
      out[i].dy = m.cells[i].dy;
      out[i].dx = m.cells[i].dx;
    }
  });
}

int ref_scatter_gather(const float* blocks, int count, int block, const int32_t* prod_idx,
                       const float* orig_out, int n, int c, int h, int w,
                       const int32_t* cons_idx, int cons_count, int cons_block, int ch, int cw,
                       int k, int s, const sige_epilogue* epi, float* out) {
  return guarded([&] {
    BlockIndexSet prod = to_index_set(prod_idx, count, block, h, w);
    BlockStack bs = to_stack(blocks, count, c, block, 0, prod);
    ScatterMap map = build_scatter_map(prod);
    BlockStack g = scatter_gather(bs, to_tensor(orig_out, n, c, h, w), map,
                                  to_index_set(cons_idx, cons_count, cons_block, ch, cw), k, s,
                                  to_epilogue(epi));
    std::memcpy(out, g.data.data(), g.data.size() * sizeof(float));
  });
}

int ref_scatter_with_block_residual(const float* mb, int mcount, int mblock, const int32_t* midx,
                                    const float* sb, int scount, int sblock, const int32_t* sidx,
                                    const float* sum, const float* orig_sc, float* out, int n,
                                    int c, int h, int w, int fused) {
  return guarded([&] {
    BlockStack m = to_stack(mb, mcount, c, mblock, 0, to_index_set(midx, mcount, mblock, h, w));
    BlockStack s = to_stack(sb, scount, c, sblock, 0, to_index_set(sidx, scount, sblock, h, w));
    Tensor ts = to_tensor(sum, n, c, h, w), to = to_tensor(orig_sc, n, c, h, w);
    from_tensor(fused ? scatter_with_block_residual(m, s, ts, to)
                      : scatter_with_block_residual_unfused(m, s, ts, to),
                out);
  });
}

int ref_apply_epilogue_on_blocks(float* blocks, int count, int channels, int bh,
                                 const int32_t* idx, int idx_h, int idx_w,
                                 const sige_epilogue* epi) {
  return guarded([&] {
    BlockStack s = to_stack(blocks, count, channels, bh, 0, to_index_set(idx, count, bh, idx_h, idx_w));
    apply_epilogue_on_blocks(s, to_epilogue(epi));
    std::memcpy(blocks, s.data.data(), s.data.size() * sizeof(float));
  });
}

int ref_conv_on_blocks(const float* blocks, int count, int window, const sige_conv_desc* conv,
                       int with_bias, float* out, int block) {
  return guarded([&] {
    ConvLayer L = to_conv(*conv);
    BlockIndexSet dummy;
    dummy.block_size = block;
    dummy.indices.resize(count);
    BlockStack in = to_stack(blocks, count, conv->c_in, block, window - block, dummy);
    BlockStack o = conv_on_blocks(in, L, with_bias != 0);
    std::memcpy(out, o.data.data(), o.data.size() * sizeof(float));
  });
}

int ref_conv2d(const float* x, int n, int c, int h, int w, const sige_conv_desc* conv,
               int with_bias, float* out) {
  return guarded([&] { from_tensor(conv2d(to_tensor(x, n, c, h, w), to_conv(*conv), with_bias != 0), out); });
}

int ref_group_norm_fold(const float* x, int n, int c, int h, int w, int groups, float eps,
                        const float* gamma, const float* beta, float* scale, float* shift) {
  return guarded([&] {
    NormStats st = compute_norm_stats(to_tensor(x, n, c, h, w), groups, eps);
    FoldedNorm f = fold_stats(st, std::vector<float>(gamma, gamma + c),
                              std::vector<float>(beta, beta + c), c);
    std::memcpy(scale, f.scale.data(), f.scale.size() * sizeof(float));
    std::memcpy(shift, f.shift.data(), f.shift.size() * sizeof(float));
  });
}

// ---- models, cache, executor -------------------------------------------

void* ref_model_build(const char* name) {
  ModelSpec* m = nullptr;
  int rc = guarded([&] { m = new ModelSpec(build_named(name)); });
  return rc == 0 ? m : nullptr;
}

void* ref_model_from_desc(const sige_model_desc* d) {
  ModelSpec* out = nullptr;
  int rc = guarded([&] {
    auto m = std::make_unique<ModelSpec>();
    m->name = d->name ? d->name : "";
    m->in_channels = d->in_channels;
    m->in_h = d->in_h;
    m->in_w = d->in_w;
    for (int i = 0; i < d->num_layers; ++i) {
      const sige_layer_desc& ld = d->layers[i];
      Layer L;
      L.kind = static_cast<LayerKind>(ld.kind);
      L.name = "l" + std::to_string(i);
      L.policy.sparse = ld.policy_sparse != 0;
      L.policy.min_resolution = ld.min_resolution;
      switch (L.kind) {
        case LayerKind::Conv:
        case LayerKind::Downsample:
          L.conv = to_conv(ld.conv);
          break;
        case LayerKind::Norm:
          L.norm = to_norm(ld.norm);
          break;
        case LayerKind::Activation:
          L.act = static_cast<ActKind>(ld.act);
          break;
        case LayerKind::ResBlock:
          L.res.conv1 = to_conv(ld.conv);
          L.res.conv2 = to_conv(ld.conv2);
          L.res.norm = to_norm(ld.norm);
          L.res.act = static_cast<ActKind>(ld.act);
          if (ld.has_shortcut) L.res.shortcut = to_conv(ld.shortcut);
          break;
        case LayerKind::Upsample:
          break;
      }
      m->layers.push_back(std::move(L));
    }
    m->validate();
    out = m.release();
  });
  return rc == 0 ? out : nullptr;
}

void ref_model_free(void* m) { delete static_cast<ModelSpec*>(m); }

uint64_t ref_model_weight_hash(void* m) { return model_weight_hash(*static_cast<ModelSpec*>(m)); }
uint64_t ref_model_structure_hash(void* m) { return static_cast<ModelSpec*>(m)->structure_hash(); }

int ref_model_required_dilation(void* m) { return required_dilation(*static_cast<ModelSpec*>(m)); }

int ref_model_output_shape(void* m, int* c, int* h, int* w) {
  return guarded([&] {
    ModelSpec& ms = *static_cast<ModelSpec*>(m);
    auto shapes = walk_shapes(ms, ms.in_h, ms.in_w);
    *c = shapes.back().c_out;
    *h = shapes.back().h_out;
    *w = shapes.back().w_out;
  });
}

// Layer-by-layer dump of the model as sige_layer_desc rows is not needed:
// tests compare weight hashes and outputs.

void* ref_cache_precompute(void* model, const float* orig, int n, int c, int h, int w,
                           int keep_inputs) {
  ActivationCache* cache = nullptr;
  int rc = guarded([&] {
    auto cc = std::make_unique<ActivationCache>();
    PrecomputeOptions opts;
    opts.keep_conv_inputs = keep_inputs != 0;
    precompute(*cc, *static_cast<ModelSpec*>(model), to_tensor(orig, n, c, h, w), {0}, opts);
    cache = cc.release();
  });
  return rc == 0 ? cache : nullptr;
}

void ref_cache_free(void* c) { delete static_cast<ActivationCache*>(c); }

int ref_cache_tensor(void* cache, int step, const char* key, float* out, size_t cap, int* dims) {
  return guarded([&] {
    const Tensor& t = static_cast<ActivationCache*>(cache)->tensor_entry(step, key);
    dims[0] = t.n;
    dims[1] = t.c;
    dims[2] = t.h;
    dims[3] = t.w;
    if (out && cap >= t.numel()) from_tensor(t, out);
  });
}

int ref_cache_norm(void* cache, int step, const char* key, float* scale, float* shift,
                   size_t cap, int* count) {
  return guarded([&] {
    const FoldedNorm& f = static_cast<ActivationCache*>(cache)->norm_entry(step, key);
    *count = static_cast<int>(f.scale.size());
    if (scale && cap >= f.scale.size()) {
      std::memcpy(scale, f.scale.data(), f.scale.size() * sizeof(float));
      std::memcpy(shift, f.shift.data(), f.shift.size() * sizeof(float));
    }
  });
}

uint64_t ref_cache_total_elements(void* cache) {
  return static_cast<ActivationCache*>(cache)->total_elements();
}

int ref_sparse_forward(void* model, void* cache, const float* edited, int n, int c, int h, int w,
                       const uint8_t* mask, const sige_run_config* cfg, float* out,
                       uint64_t* trace_rows, int trace_cap, int* trace_n) {
  return guarded([&] {
    RunTrace tr;
    Tensor o = sparse_forward(*static_cast<ModelSpec*>(model), to_tensor(edited, n, c, h, w),
                              *static_cast<ActivationCache*>(cache), to_mask(mask, h, w),
                              to_config(cfg), &tr);
    from_tensor(o, out);
    write_trace(tr, trace_rows, trace_cap, trace_n);
  });
}

int ref_dense_forward(void* model, const float* in, int n, int c, int h, int w, float* out) {
  return guarded([&] {
    from_tensor(dense_forward(*static_cast<ModelSpec*>(model), to_tensor(in, n, c, h, w)), out);
  });
}

int ref_dense_forward_reused_stats(void* model, const float* in, int n, int c, int h, int w,
                                   void* cache, int step, float* out) {
  return guarded([&] {
    from_tensor(dense_forward_reused_stats(*static_cast<ModelSpec*>(model),
                                           to_tensor(in, n, c, h, w),
                                           *static_cast<ActivationCache*>(cache), step),
                out);
  });
}

int ref_output_coverage(void* model, const uint8_t* mask, int h, int w, int batch,
                        const sige_run_config* cfg, uint8_t* out, int* oh, int* ow) {
  return guarded([&] {
    DifferenceMask cov = output_coverage(*static_cast<ModelSpec*>(model), to_mask(mask, h, w),
                                         batch, to_config(cfg));
    *oh = cov.h;
    *ow = cov.w;
    if (out) std::memcpy(out, cov.bits.data(), cov.bits.size());
  });
}

}  // extern "C"

// Cache construction through the reference's public ActivationCache API
// (graph.hpp:116-156) — lets bench.py's CPU baseline skip the (untimed)
// dense precompute by seeding the reference cache with already computed
// entries.
extern "C" {

void* ref_cache_create_for(void* model) {
  auto* c = new ActivationCache();
  c->set_model_hash(static_cast<ModelSpec*>(model)->structure_hash());
  return c;
}

int ref_cache_put_tensor(void* cache, int step, const char* key, const float* data, int n, int c,
                         int h, int w) {
  return guarded([&] {
    static_cast<ActivationCache*>(cache)->put_tensor(step, key, to_tensor(data, n, c, h, w),
                                                     CacheCategory::ConvOutput);
  });
}

int ref_cache_put_norm(void* cache, int step, const char* key, const float* scale,
                       const float* shift, int count) {
  return guarded([&] {
    FoldedNorm f;
    f.scale.assign(scale, scale + count);
    f.shift.assign(shift, shift + count);
    static_cast<ActivationCache*>(cache)->put_norm(step, key, std::move(f));
  });
}

}  // extern "C"

#ifdef SIGE_REF_IO
// On-disk formats through the reference's own io.cpp (io.hpp:12-36): the
// tests exchange files both ways with the library's sige_save_* / sige_load_*.
extern "C" {

int ref_io_save_tensor(const char* path, const float* x, int n, int c, int h, int w) {
  return guarded([&] { save_tensor(path, to_tensor(x, n, c, h, w)); });
}

int ref_io_load_tensor(const char* path, float* out, size_t cap, int* dims) {
  return guarded([&] {
    Tensor t = load_tensor(path);
    dims[0] = t.n, dims[1] = t.c, dims[2] = t.h, dims[3] = t.w;
    if (out && cap >= t.data.size()) from_tensor(t, out);
  });
}

int ref_io_save_mask_pbm(const char* path, const uint8_t* m, int h, int w) {
  return guarded([&] { save_mask_pbm(path, to_mask(m, h, w)); });
}

int ref_io_load_mask_pbm(const char* path, uint8_t* out, size_t cap, int* h, int* w) {
  return guarded([&] {
    DifferenceMask m = load_mask_pbm(path);
    *h = m.h, *w = m.w;
    if (out && cap >= m.bits.size()) std::memcpy(out, m.bits.data(), m.bits.size());
  });
}

int ref_io_save_block_stack(const char* prefix, const float* data, int count, int channels, int block, int overlap,
                            int origin_block, int origin_h, int origin_w, const int32_t* idx) {
  return guarded([&] {
    BlockStack st;
    st.channels = channels;
    st.block = block;
    st.overlap = overlap;
    st.origin = to_index_set(idx, count, origin_block, origin_h, origin_w);
    st.data.assign(data, data + static_cast<size_t>(count) * channels * (block + overlap) * (block + overlap));
    save_block_stack(prefix, st);
  });
}

int ref_io_load_block_stack(const char* prefix, float* data, size_t cap, int32_t* idx, size_t idx_cap, int* meta) {
  return guarded([&] {
    BlockStack st = load_block_stack(prefix);
    meta[0] = static_cast<int>(st.count()), meta[1] = st.channels, meta[2] = st.block, meta[3] = st.overlap;
    meta[4] = st.origin.block_size, meta[5] = st.origin.h, meta[6] = st.origin.w;
    if (data && cap >= st.data.size()) std::memcpy(data, st.data.data(), st.data.size() * sizeof(float));
    if (idx && idx_cap >= 3 * st.count())
      for (size_t g = 0; g < st.count(); ++g) {
        idx[3 * g] = st.origin.indices[g].n;
        idx[3 * g + 1] = st.origin.indices[g].r;
        idx[3 * g + 2] = st.origin.indices[g].c;
      }
  });
}

}  // extern "C"
#endif  // SIGE_REF_IO
