// capi.cpp — the extern "C" boundary declared in include/sige_b200.h.
// Every entry point validates like the reference (ConfigError messages with
// the reference's op prefixes), converts exceptions into status codes and
// keeps the message in a thread-local for sige_last_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "common.hpp"
#include "engine.hpp"
#include "models.hpp"
#include "ops.hpp"
#include "sige_b200.h"

using namespace sige_b200;

namespace sige_b200 {  // io.cpp
void io_write_sigt(const std::string& path, const uint32_t d[4], const float* data);
void io_read_sigt(const std::string& path, uint32_t d[4], float* out, size_t cap);
void io_save_mask_pbm(const std::string& path, const uint8_t* m, int h, int w);
void io_load_mask_pbm(const std::string& path, int* h, int* w, uint8_t* out, size_t cap);
void io_save_block_stack(const std::string& prefix, const float* data, int count, int channels, int block,
                         int overlap, int origin_block, int origin_h, int origin_w, const int32_t* idx);
void io_load_block_stack(const std::string& prefix, int meta[7], float* data, size_t cap, int32_t* idx,
                         size_t idx_cap);
}  // namespace sige_b200

// Device staging of the host-buffer entry point, owned by the engine handle
// (freed in sige_engine_destroy).
struct HostStage {
  float* d_in = nullptr;
  float* d_out = nullptr;
  uint8_t* d_mask = nullptr;
  size_t in_n = 0, out_n = 0, mask_n = 0;
  ~HostStage() {
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_mask);
  }
};

struct sige_engine {
  Engine* impl;
  HostStage stage;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SIGE_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return SIGE_ERR_CONFIG;
  } catch (const CudaError& e) {
    g_err = e.what();
    return SIGE_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SIGE_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw ConfigError(std::string(what) + ": null pointer");
}

// Scratch device buffer for small temporaries of op-level calls.
template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { SIGE_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T))); }
  ~DevBuf() { cudaFree(p); }
};

}  // namespace

extern "C" {

const char* sige_last_error(void) { return g_err.c_str(); }
const char* sige_version(void) { return "sige_b200 0.1 (sm_100a)"; }
uint64_t sige_kernel_launch_count(void) { return g_launches.load(); }

// Developer instrumentation, not part of the reference-facing ABI: per-launch
// [start, end] globaltimer of k_conv_tc launches when SIGE_TC_GTL=1.
int sige_debug_conv_timeline(unsigned long long* out, int cap) { return sige_b200::debug_conv_timeline(out, cap); }
int sige_debug_conv_marks(unsigned long long* out, int cap) { return sige_b200::debug_conv_marks(out, cap); }
// Device glibc expf (mode 0) / exact SiLU (mode 1) of the float bit patterns
// first .. first+count-1, with the libm build the host dispatches to.
int sige_debug_expf_sweep(uint32_t first, long long count, int mode, float* out, sige_stream_t s) {
  return guarded([&] {
    if (mode != 0 && mode != 1) throw ConfigError("expf_sweep: mode must be 0 (expf) or 1 (silu)");
    op_expf_sweep(first, count, mode, out, as_stream(s));
  });
}
int sige_debug_host_expf_is_fma(void) { return sige_b200::host_expf_is_fma() ? 1 : 0; }

void sige_run_config_default(sige_run_config* c) {  // graph.hpp:87-101
  c->step = 0;
  c->mask_threshold = 1e-3f;
  c->dilate_full = 1;
  c->dilate_scale = 1;
  c->block3 = 6;
  c->block1 = 4;
  c->min_sparse_res = -1;
  c->sparse = 1;
  c->norm_precompute = 1;
  c->elem_fusion = 1;
  c->scatter_fusion = 1;
  c->seed = 42;
}

int sige_compute_difference_mask(const float* original, const float* edited, int n, int c, int h,
                                 int w, float threshold, uint8_t* mask_out, sige_stream_t s) {
  return guarded([&] {
    need(original, "compute_difference_mask");
    need(edited, "compute_difference_mask");
    need(mask_out, "compute_difference_mask");
    op_difference_mask(original, edited, n, c, h, w, threshold, mask_out, as_stream(s));
  });
}

int sige_downsample_mask(const uint8_t* mask, int h, int w, int out_h, int out_w, uint8_t* out,
                         sige_stream_t s) {
  return guarded([&] { op_downsample_mask(mask, h, w, out_h, out_w, out, as_stream(s)); });
}

int sige_dilate_mask(const uint8_t* mask, int h, int w, int radius, uint8_t* out, sige_stream_t s) {
  return guarded([&] {
    if (radius < 0) throw ConfigError("dilate_mask: radius must be >= 0");
    DevBuf<uint8_t> tmp(static_cast<size_t>(h) * w);
    op_dilate_mask(mask, h, w, radius, out, tmp.p, as_stream(s));
    SIGE_CUDA(cudaStreamSynchronize(as_stream(s)));
  });
}

int sige_mask_to_block_indices_async(const uint8_t* mask, int h, int w, int block_size, int batch,
                                     int32_t* indices, int capacity, int32_t* count_device,
                                     sige_stream_t s) {
  return guarded([&] {
    op_mask_to_block_indices(mask, h, w, block_size, batch, indices, capacity, count_device,
                             as_stream(s));
  });
}

int sige_mask_to_block_indices(const uint8_t* mask, int h, int w, int block_size, int batch,
                               int32_t* indices, int capacity, int* count_host, sige_stream_t s) {
  return guarded([&] {
    DevBuf<int32_t> cnt(1);
    op_mask_to_block_indices(mask, h, w, block_size, batch, indices, capacity, cnt.p, as_stream(s));
    int32_t v = 0;
    SIGE_CUDA(cudaMemcpyAsync(&v, cnt.p, sizeof v, cudaMemcpyDeviceToHost, as_stream(s)));
    SIGE_CUDA(cudaStreamSynchronize(as_stream(s)));
    *count_host = v;
  });
}

int sige_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count,
                int block_size, int idx_h, int idx_w, int k, int stride,
                const sige_epilogue* epilogue, float* out, sige_stream_t s) {
  return guarded([&] {
    DevEpilogue e = make_dev_epilogue(epilogue, c, n);
    op_gather(x, n, c, h, w, idx, count, block_size, idx_h, idx_w, k, stride, e, out, as_stream(s));
  });
}

int sige_gather_spade(const float* x, const float* gamma, const float* beta, int n, int c, int h, int w,
                      const int32_t* idx, int count, int block, int idx_h, int idx_w, int k, int stride,
                      const sige_epilogue* norm, int act, float* out, sige_stream_t s) {
  return guarded([&] {
    if (count) {
      need(x, "gather_spade");
      need(gamma, "gather_spade");
      need(beta, "gather_spade");
    }
    DevEpilogue e = make_dev_epilogue(norm, c, n);
    op_gather_spade(x, gamma, beta, n, c, h, w, idx, count, block, idx_h, idx_w, k, stride, e, act, out,
                    as_stream(s));
  });
}

int sige_resize_nearest(const float* in, int n, int c, int h, int w, int out_h, int out_w, float* out,
                        sige_stream_t s) {
  return guarded([&] { op_resize_nearest(in, n, c, h, w, out_h, out_w, out, as_stream(s)); });
}


int sige_scatter_inplace(const float* blocks, int count, int channels, int block, const int32_t* idx,
                         float* base, int n, int c, int h, int w, sige_stream_t s) {
  return guarded([&] { op_scatter(blocks, count, channels, block, idx, base, n, c, h, w, false, as_stream(s)); });
}

int sige_scatter(const float* blocks, int count, int channels, int block, const int32_t* idx,
                 const float* base, float* out, int n, int c, int h, int w, sige_stream_t s) {
  return guarded([&] {
    if (out != base)
      SIGE_CUDA(cudaMemcpyAsync(out, base, sizeof(float) * n * c * h * w, cudaMemcpyDeviceToDevice,
                                as_stream(s)));
    op_scatter(blocks, count, channels, block, idx, out, n, c, h, w, false, as_stream(s));
  });
}

int sige_scatter_add_inplace(const float* blocks, int count, int channels, int block,
                             const int32_t* idx, float* base, int n, int c, int h, int w,
                             sige_stream_t s) {
  return guarded([&] { op_scatter(blocks, count, channels, block, idx, base, n, c, h, w, true, as_stream(s)); });
}

int sige_build_scatter_map(const int32_t* idx, int count, int block, int h, int w,
                           sige_scatter_entry* map_out, int* bps, sige_stream_t s) {
  return guarded([&] {
    DevBuf<int> scratch(2);
    *bps = op_build_scatter_map(idx, count, block, h, w, map_out, scratch.p, as_stream(s));
  });
}

namespace {
// BlockIndexSet::content_hash (mask.cpp:91-101) of a device index set.
uint64_t index_set_hash(const int32_t* idx, int count, int block, int h, int w, cudaStream_t st) {
  std::vector<int32_t> host(static_cast<size_t>(count) * 3);
  if (count) {
    SIGE_CUDA(cudaMemcpyAsync(host.data(), idx, host.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SIGE_CUDA(cudaStreamSynchronize(st));
  }
  uint64_t hs = fnv1a64(&block, sizeof(block));
  hs = fnv1a64(&h, sizeof(h), hs);
  hs = fnv1a64(&w, sizeof(w), hs);
  for (int i = 0; i < count; ++i)
    for (int j = 0; j < 3; ++j) hs = fnv1a64(&host[3 * i + j], sizeof(int32_t), hs);
  return hs;
}

// ScatterMapCache (kernels.hpp:80-91, kernels.cpp:171-202) on the device: one
// scatter map per index-set content hash, built once and kept until clear().
struct MapEntry {
  sige_scatter_entry* map = nullptr;
  int bps = 0;
};
std::mutex g_map_mu;
std::unordered_map<uint64_t, MapEntry> g_maps;
}  // namespace

int sige_block_index_hash(const int32_t* idx, int count, int block, int h, int w, uint64_t* out, sige_stream_t s) {
  return guarded([&] {
    need(out, "content_hash");
    *out = index_set_hash(idx, count, block, h, w, as_stream(s));
  });
}

int sige_scatter_map_cache_get(const int32_t* idx, int count, int block, int h, int w,
                               const sige_scatter_entry** map_out, int* bps, uint64_t* key_out, sige_stream_t s) {
  return guarded([&] {
    need(map_out, "ScatterMapCache::get");
    need(bps, "ScatterMapCache::get");
    cudaStream_t st = as_stream(s);
    const uint64_t key = index_set_hash(idx, count, block, h, w, st);
    if (key_out) *key_out = key;
    std::lock_guard<std::mutex> lock(g_map_mu);
    auto it = g_maps.find(key);
    if (it == g_maps.end()) {
      MapEntry e;
      SIGE_CUDA(cudaMalloc(&e.map, std::max<size_t>(static_cast<size_t>(h) * w, 1) * sizeof(sige_scatter_entry)));
      try {
        DevBuf<int> scratch(2);
        e.bps = op_build_scatter_map(idx, count, block, h, w, e.map, scratch.p, st);
      } catch (...) {
        cudaFree(e.map);
        throw;
      }
      it = g_maps.emplace(key, e).first;
    }
    *map_out = it->second.map;
    *bps = it->second.bps;
  });
}

size_t sige_scatter_map_cache_size(void) {
  std::lock_guard<std::mutex> lock(g_map_mu);
  return g_maps.size();
}

void sige_scatter_map_cache_clear(void) {
  std::lock_guard<std::mutex> lock(g_map_mu);
  cudaDeviceSynchronize();  // maps may still be read by queued scatter_gather launches
  for (auto& kv : g_maps) cudaFree(kv.second.map);
  g_maps.clear();
}

int sige_scatter_gather(const float* blocks, int count, int block, const float* original_out, int n,
                        int c, int h, int w, const sige_scatter_entry* map, int blocks_per_sample,
                        const int32_t* consumer_idx, int consumer_count, int consumer_block,
                        int consumer_h, int consumer_w, int k, int stride,
                        const sige_epilogue* epilogue, float* out, sige_stream_t s) {
  return guarded([&] {
    DevEpilogue e = make_dev_epilogue(epilogue, c, n);
    op_scatter_gather(blocks, count, block, original_out, n, c, h, w, map, blocks_per_sample,
                      consumer_idx, consumer_count, consumer_block, consumer_h, consumer_w, k,
                      stride, e, out, as_stream(s));
  });
}

int sige_scatter_with_block_residual(const float* mb, int mcount, int mblock, const int32_t* midx,
                                     const float* sb, int scount, int sblock, const int32_t* sidx,
                                     const float* sum, const float* orig_sc, float* out, int n,
                                     int c, int h, int w, sige_stream_t s) {
  return guarded([&] {
    cudaStream_t st = as_stream(s);
    SIGE_CUDA(cudaMemcpyAsync(out, sum, sizeof(float) * n * c * h * w, cudaMemcpyDeviceToDevice, st));
    op_residual_pass(mb, mcount, c, mblock, midx, orig_sc, out, n, h, w, false, st);
    op_residual_pass(sb, scount, c, sblock, sidx, orig_sc, out, n, h, w, true, st);
  });
}

int sige_scatter_with_block_residual_unfused(const float* mb, int mcount, int mblock,
                                             const int32_t* midx, const float* sb, int scount,
                                             int sblock, const int32_t* sidx, const float* sum,
                                             const float* orig_sc, float* out, int n, int c, int h,
                                             int w, sige_stream_t s) {
  // kernels.cpp:339-355: gather(orig_sc) -> add -> scatter; gather -> subtract -> scatter_add.
  return guarded([&] {
    cudaStream_t st = as_stream(s);
    SIGE_CUDA(cudaMemcpyAsync(out, sum, sizeof(float) * n * c * h * w, cudaMemcpyDeviceToDevice, st));
    DevEpilogue none = make_dev_epilogue(nullptr, c, n);
    size_t mz = static_cast<size_t>(mcount) * c * mblock * mblock;
    size_t sz = static_cast<size_t>(scount) * c * sblock * sblock;
    DevBuf<float> g(std::max(mz, sz)), t(std::max(mz, sz));
    op_gather(orig_sc, n, c, h, w, midx, mcount, mblock, h, w, 1, 1, none, g.p, st);
    op_combine(mb, g.p, 1.0f, mz, t.p, st);
    op_scatter(t.p, mcount, c, mblock, midx, out, n, c, h, w, false, st);
    op_gather(orig_sc, n, c, h, w, sidx, scount, sblock, h, w, 1, 1, none, g.p, st);
    op_combine(sb, g.p, -1.0f, sz, t.p, st);
    op_scatter(t.p, scount, c, sblock, sidx, out, n, c, h, w, true, st);
    SIGE_CUDA(cudaStreamSynchronize(st));
  });
}

int sige_combine_blocks(const float* a, const float* b, float sign, size_t numel, float* out,
                        sige_stream_t s) {
  return guarded([&] { op_combine(a, b, sign, numel, out, as_stream(s)); });
}

int sige_apply_epilogue_on_blocks(float* blocks, int count, int channels, int bh,
                                  const int32_t* idx, const sige_epilogue* epilogue,
                                  sige_stream_t s) {
  return guarded([&] {
    // per-sample params are indexed by each block's own n (eltwise.cpp:48-58)
    DevEpilogue e = make_dev_epilogue(epilogue, channels, 1);
    op_epilogue_blocks(blocks, count, channels, bh, idx, e, as_stream(s));
  });
}

namespace {
void check_math_mode(int m, const char* op) {
  if (m != SIGE_MATH_EXACT && m != SIGE_MATH_FP32_FMA && m != SIGE_MATH_TF32 && m != SIGE_MATH_F16)
    throw ConfigError(std::string(op) + ": unknown math mode " + std::to_string(m));
}

// RAII device scratch of an op-level call (freed after the stream drains).
struct Scratch {
  std::vector<void*> ptrs;
  cudaStream_t st;
  explicit Scratch(cudaStream_t s) : st(s) {}
  void* get(size_t bytes) {
    void* p = nullptr;
    SIGE_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    ptrs.push_back(p);
    return p;
  }
  ~Scratch() {
    cudaStreamSynchronize(st);
    for (void* p : ptrs) cudaFree(p);
  }
};

// Op-level conv on the tcgen05 tensor cores (SIGE_MATH_F16 / SIGE_MATH_TF32):
// the NCHW fp32 source `x` (n, c, h, w) is convolved over the output tile list
// `tiles` (origins at output resolution) with padding `pad` by the engine's
// fused kernel (launch_conv_tc) into an NHWC scratch, then written to `out`
// (NCHW, n x c_out x oh x ow). The weights are packed per call.
void op_conv_tc(const float* x, int n, int c, int h, int w, const sige_conv_desc& cv, bool with_bias,
                int math, int pad, const std::vector<int32_t>& tiles_host, int bh, int bw, int oh, int ow,
                float* out, cudaStream_t st) {
  Scratch S(st);
  const bool f16 = math == SIGE_MATH_F16;
  ConvW cw;
  cw.c_in = cv.c_in;
  cw.c_out = cv.c_out;
  cw.k = cv.k;
  cw.stride = cv.stride;
  cw.w = cv.weight;
  cw.bias = with_bias ? cv.bias : nullptr;
  pack_weights_tc(cv.weight, cv.c_out, cv.c_in, cv.k, f16 ? 1 : 0, &cw, st);
  S.ptrs.push_back(const_cast<void*>(cw.w_tc));
  Src src;
  src.ptr = x;
  src.layout = kNCHW;
  src.n = n;
  src.c = c;
  src.h = h;
  src.w = w;
  src.epi.fma_expf = host_expf_is_fma() ? 1 : 0;
  Tiles t;
  int32_t* idx = static_cast<int32_t*>(S.get(tiles_host.size() * sizeof(int32_t)));
  SIGE_CUDA(cudaMemcpyAsync(idx, tiles_host.data(), tiles_host.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  t.idx = idx;
  t.count = static_cast<int>(tiles_host.size() / 3);
  t.capacity = t.count;
  t.bh = bh;
  t.bw = bw;
  float* tmp = static_cast<float*>(S.get(static_cast<size_t>(n) * oh * ow * cv.c_out * sizeof(float)));
  Dst d;
  d.ptr = tmp;
  d.n = n;
  d.c = cv.c_out;
  d.h = oh;
  d.w = ow;
  d.mode = kStore;
  launch_conv_tc(src, t, cw, d, f16 ? 1 : 0, st, 0, nullptr, 0, pad);
  Src r;
  r.ptr = tmp;
  r.layout = kNHWC;
  r.n = n;
  r.c = cv.c_out;
  r.h = oh;
  r.w = ow;
  launch_materialize(r, out, kNCHW, st);
}
}  // namespace

int sige_conv_on_blocks(const float* blocks, int count, int window, const sige_conv_desc* conv,
                        int with_bias, int math_mode, float* out, int block, sige_stream_t s) {
  return guarded([&] {
    need(conv, "conv_on_blocks");
    check_math_mode(math_mode, "conv_on_blocks");
    const sige_conv_desc& cv = *conv;
    if (cv.k != 1 && cv.k != 3) throw ConfigError("conv: kernel size must be 1 or 3, got " + std::to_string(cv.k));
    if (cv.stride != 1 && cv.stride != 2)
      throw ConfigError("conv: stride must be 1 or 2, got " + std::to_string(cv.stride));
    int b_out = (window - cv.k) / cv.stride + 1;  // kernels.cpp:397-405
    if (b_out != block)
      throw ConfigError("conv_on_blocks: window " + std::to_string(window) + " with k=" +
                        std::to_string(cv.k) + " s=" + std::to_string(cv.stride) + " yields " +
                        std::to_string(b_out) + ", expected block " + std::to_string(block));
    if (count == 0) return;
    if (math_mode == SIGE_MATH_TF32 || math_mode == SIGE_MATH_F16) {
      // one tile per block: the block stack is an NCHW batch of count windows,
      // each convolved without padding (the gather carried the halo)
      std::vector<int32_t> tiles(static_cast<size_t>(count) * 3, 0);
      for (int g = 0; g < count; ++g) tiles[3 * g] = g;
      op_conv_tc(blocks, count, cv.c_in, window, window, cv, with_bias != 0, math_mode, 0, tiles, block, block,
                 block, block, out, as_stream(s));
      return;
    }
    op_conv_cc(blocks, static_cast<long long>(cv.c_in) * window * window, cv.c_in, window, window,
               cv.weight, with_bias ? cv.bias : nullptr, cv.c_out, cv.k, cv.stride, 0, out,
               static_cast<long long>(cv.c_out) * block * block, block, block, count, math_mode,
               as_stream(s));
  });
}

int sige_conv2d(const float* x, int n, int c, int h, int w, const sige_conv_desc* conv, int with_bias,
                int math_mode, float* out, sige_stream_t s) {
  return guarded([&] {
    need(conv, "conv2d");
    check_math_mode(math_mode, "conv2d");
    const sige_conv_desc& cv = *conv;
    if (c != cv.c_in)
      throw ConfigError("conv2d: input has " + std::to_string(c) + " channels, layer expects " +
                        std::to_string(cv.c_in));
    int oh = conv_out_dim(h, cv.k, cv.stride), ow = conv_out_dim(w, cv.k, cv.stride);
    if (math_mode == SIGE_MATH_TF32 || math_mode == SIGE_MATH_F16) {
      if (cv.k != 1 && cv.k != 3) throw ConfigError("conv: kernel size must be 1 or 3, got " + std::to_string(cv.k));
      if (cv.stride != 1 && cv.stride != 2)
        throw ConfigError("conv: stride must be 1 or 2, got " + std::to_string(cv.stride));
      if (n == 0 || oh <= 0 || ow <= 0) return;
      // output tiles as the engine's dense pass lays them out (one M=128 MMA each)
      const int bw = std::min(ow, 16);
      const int P = cv.stride == 1 ? bw + cv.k - 1 : bw + 1;
      const int bh = std::max(1, std::min(oh, (128 - bw) / P + 1));
      std::vector<int32_t> tiles;
      for (int i = 0; i < n; ++i)
        for (int r = 0; r < oh; r += bh)
          for (int q = 0; q < ow; q += bw) tiles.insert(tiles.end(), {i, r, q});
      op_conv_tc(x, n, c, h, w, cv, with_bias != 0, math_mode, (cv.k - 1) / 2, tiles, bh, bw, oh, ow, out,
                 as_stream(s));
      return;
    }
    op_conv_cc(x, static_cast<long long>(c) * h * w, c, h, w, cv.weight, with_bias ? cv.bias : nullptr,
               cv.c_out, cv.k, cv.stride, (cv.k - 1) / 2, out,
               static_cast<long long>(cv.c_out) * oh * ow, oh, ow, n, math_mode, as_stream(s));
  });
}

// ---- engine
int sige_engine_create(const sige_model_desc* model, int batch, int math_mode, sige_engine** out) {
  return guarded([&] {
    need(model, "engine");
    need(out, "engine");
    *out = new sige_engine{new Engine(model, batch, math_mode)};
  });
}

void sige_engine_destroy(sige_engine* eng) {
  if (!eng) return;
  delete eng->impl;  // synchronises the device before freeing
  delete eng;
}

int sige_engine_precompute(sige_engine* eng, const float* original, int step, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    need(original, "precompute");
    eng->impl->precompute(original, step, as_stream(s));
  });
}

int sige_engine_output_coverage(sige_engine* eng, const float* edited, const uint8_t* mask,
                                const sige_run_config* cfg, uint8_t* out, int* out_h, int* out_w, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    need(out, "output_coverage");
    if (!edited && !mask) throw ConfigError("output_coverage: needs the edited input or a mask");
    sige_run_config c;
    if (cfg)
      c = *cfg;
    else
      sige_run_config_default(&c);
    int oh = 0, ow = 0;
    eng->impl->output_coverage(edited, mask, c, out, &oh, &ow, as_stream(s));
    if (out_h) *out_h = oh;
    if (out_w) *out_w = ow;
  });
}

int sige_engine_offload_step(sige_engine* eng, int step, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    eng->impl->offload_step(step, as_stream(s));
  });
}

int sige_engine_prefetch_step(sige_engine* eng, int step, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    eng->impl->prefetch_step(step, as_stream(s));
  });
}

int sige_engine_drop_step(sige_engine* eng, int step) {
  return guarded([&] {
    need(eng, "engine");
    eng->impl->drop_step(step);
  });
}

int sige_engine_refresh_step(sige_engine* eng, const float* original, int step, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    need(original, "refresh_step");
    eng->impl->refresh_step(original, step, as_stream(s));
  });
}

int sige_engine_cache_model_hash(const sige_engine* eng, uint64_t* cache_hash, uint64_t* model_hash) {
  return guarded([&] {
    need(eng, "engine");
    if (cache_hash) *cache_hash = eng->impl->cache_model_hash();
    if (model_hash) *model_hash = eng->impl->structure_hash();
  });
}

int sige_engine_set_cache_model_hash(sige_engine* eng, uint64_t cache_hash) {
  return guarded([&] {
    need(eng, "engine");
    eng->impl->set_cache_model_hash(cache_hash);
  });
}

uint64_t sige_model_structure_hash(const sige_model_desc* model) {
  return model ? sige_b200::model_structure_hash(model) : 0;
}

int sige_engine_put_tensor(sige_engine* eng, int step, const char* key, const float* host,
                           size_t numel) {
  return guarded([&] { eng->impl->put_tensor(step, key, host, numel); });
}

int sige_engine_put_norm(sige_engine* eng, int step, const char* key, const float* sc,
                         const float* sh, size_t numel) {
  return guarded([&] { eng->impl->put_norm(step, key, sc, sh, numel); });
}

int sige_engine_get_tensor(sige_engine* eng, int step, const char* key, float* host, size_t numel) {
  return guarded([&] { eng->impl->get_tensor(step, key, host, numel); });
}

int sige_engine_get_norm(sige_engine* eng, int step, const char* key, float* sc, float* sh,
                         size_t numel) {
  return guarded([&] { eng->impl->get_norm(step, key, sc, sh, numel); });
}

int sige_engine_sparse_forward(sige_engine* eng, const float* edited, const uint8_t* mask,
                               const sige_run_config* cfg, float* out, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    need(edited, "sparse_forward");
    need(out, "sparse_forward");
    sige_run_config c;
    if (cfg)
      c = *cfg;
    else
      sige_run_config_default(&c);
    eng->impl->sparse_forward(edited, mask, c, out, as_stream(s));
  });
}

int sige_engine_sparse_forward_grouped(sige_engine* eng, const float* edited, const uint8_t* masks,
                                       const sige_run_config* cfg, float* out, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    need(edited, "sparse_forward");
    need(out, "sparse_forward");
    sige_run_config c;
    if (cfg)
      c = *cfg;
    else
      sige_run_config_default(&c);
    eng->impl->sparse_forward(edited, masks, c, out, as_stream(s), true);
  });
}

int sige_engine_sparse_forward_host(sige_engine* eng, const float* edited_host,
                                    const uint8_t* mask_host, const sige_run_config* cfg,
                                    float* out_host, sige_stream_t s) {
  return guarded([&] {
    need(eng, "engine");
    Engine& E = *eng->impl;
    cudaStream_t st = as_stream(s);
    int n, c, h, w;
    E.output_shape(&n, &c, &h, &w);
    const size_t in_n = static_cast<size_t>(E.batch()) * E.in_channels() * E.in_h() * E.in_w();
    const size_t out_n = static_cast<size_t>(n) * c * h * w;
    const size_t mask_n = static_cast<size_t>(E.in_h()) * E.in_w();
    HostStage& S = eng->stage;
    if (S.in_n < in_n) {
      cudaFree(S.d_in);
      SIGE_CUDA(cudaMalloc(&S.d_in, in_n * sizeof(float)));
      S.in_n = in_n;
    }
    if (S.out_n < out_n) {
      cudaFree(S.d_out);
      SIGE_CUDA(cudaMalloc(&S.d_out, out_n * sizeof(float)));
      S.out_n = out_n;
    }
    if (mask_host && S.mask_n < mask_n) {
      cudaFree(S.d_mask);
      SIGE_CUDA(cudaMalloc(&S.d_mask, mask_n));
      S.mask_n = mask_n;
    }
    SIGE_CUDA(cudaMemcpyAsync(S.d_in, edited_host, in_n * sizeof(float), cudaMemcpyHostToDevice, st));
    if (mask_host) SIGE_CUDA(cudaMemcpyAsync(S.d_mask, mask_host, mask_n, cudaMemcpyHostToDevice, st));
    sige_run_config c2;
    if (cfg)
      c2 = *cfg;
    else
      sige_run_config_default(&c2);
    E.sparse_forward(S.d_in, mask_host ? S.d_mask : nullptr, c2, S.d_out, st);
    SIGE_CUDA(cudaMemcpyAsync(out_host, S.d_out, out_n * sizeof(float), cudaMemcpyDeviceToHost, st));
    SIGE_CUDA(cudaStreamSynchronize(st));
  });
}

int sige_engine_dense_forward(sige_engine* eng, const float* input, int reused_stats, int step,
                              float* out, sige_stream_t s) {
  return guarded([&] { eng->impl->dense_forward(input, reused_stats != 0, step, out, as_stream(s)); });
}

int sige_engine_output_shape(const sige_engine* eng, int* n, int* c, int* h, int* w) {
  return guarded([&] { eng->impl->output_shape(n, c, h, w); });
}

int sige_engine_last_launch_count(const sige_engine* eng) { return eng ? eng->impl->last_launch_count() : 0; }

int sige_engine_trace(sige_engine* eng, uint64_t* rows, int cap, int* nrows, sige_stream_t s) {
  return guarded([&] { *nrows = eng->impl->trace(rows, cap, as_stream(s)); });
}

int sige_engine_set_profiling(sige_engine* eng, int enable) {
  return guarded([&] { eng->impl->set_profiling(enable != 0); });
}

int sige_engine_set_sm_budget(sige_engine* eng, int sms) {
  return guarded([&] { eng->impl->set_sm_budget(sms); });
}

int sige_engine_set_timeline(sige_engine* eng, int enable) {
  return guarded([&] { eng->impl->set_timeline(enable != 0); });
}

int sige_engine_timeline_read(sige_engine* eng, double* rows, int cap, int* nrows) {
  return guarded([&] { *nrows = eng->impl->timeline_read(rows, cap); });
}

int sige_engine_set_graphs(sige_engine* eng, int enable) {
  return guarded([&] { eng->impl->set_graphs(enable != 0); });
}

int sige_engine_profile_read(sige_engine* eng, double* rows, int cap, int* nrows, sige_stream_t s) {
  return guarded([&] { *nrows = eng->impl->profile_read(rows, cap, as_stream(s)); });
}

int sige_engine_cache_entries(const sige_engine* eng, int step, char* buf, size_t cap, size_t* needed) {
  return guarded([&] {
    std::string s = eng->impl->cache_entries(step);
    *needed = s.size() + 1;
    if (buf && cap >= s.size() + 1) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

size_t sige_engine_cache_bytes(const sige_engine* eng) { return eng ? eng->impl->cache_bytes() : 0; }

// ---- synthetic inputs
int sige_make_seg_fixture(int n, int label_nc, int h, int w, uint32_t seed, float* orig, float* edited) {
  return guarded([&] {
    if (n < 1 || label_nc < 2 || h < 8 || w < 8) throw ConfigError("seg fixture: bad shape");
    need(orig, "seg fixture");
    need(edited, "seg fixture");
    sige_b200::make_seg_fixture(n, label_nc, h, w, seed, orig, edited);
  });
}

int sige_make_edit_fixture(const char* kind, int n, int c, int h, int w, uint32_t seed,
                           float* original_host, float* edited_host) {
  return guarded([&] { make_edit_fixture(kind, n, c, h, w, seed, original_host, edited_host); });
}

int sige_model_build(const char* name, sige_model_desc** out) {
  return guarded([&] { *out = build_model(name); });
}

void sige_model_free(sige_model_desc* model) {
  if (model) free_model(model);
}

int sige_model_required_dilation(const sige_model_desc* model, int* out) {
  return guarded([&] { *out = required_dilation(model); });
}

uint64_t sige_model_weight_hash(const sige_model_desc* model) { return model_weight_hash(model); }

// ---- on-disk exchange formats (io.cpp) ----

int sige_save_tensor(const char* path, const float* host, int n, int c, int h, int w) {
  return guarded([&] {
    need(path, "save_tensor");
    if (n < 0 || c < 0 || h < 0 || w < 0) throw ConfigError("save_tensor: negative dimension");
    if (static_cast<size_t>(n) * c * h * w) need(host, "save_tensor");
    const uint32_t d[4] = {static_cast<uint32_t>(n), static_cast<uint32_t>(c), static_cast<uint32_t>(h),
                           static_cast<uint32_t>(w)};
    io_write_sigt(path, d, host);
  });
}

int sige_load_tensor(const char* path, float* host, size_t cap, int* dims) {
  return guarded([&] {
    need(path, "load_tensor");
    need(dims, "load_tensor");
    uint32_t d[4];
    io_read_sigt(path, d, nullptr, 0);
    for (uint32_t v : d)
      if (v == 0) throw ConfigError(std::string(path) + ": zero dimension");
    if (host) io_read_sigt(path, d, host, cap);
    for (int i = 0; i < 4; ++i) dims[i] = static_cast<int>(d[i]);
  });
}

int sige_save_mask_pbm(const char* path, const uint8_t* mask, int h, int w) {
  return guarded([&] {
    need(path, "save_mask_pbm");
    need(mask, "save_mask_pbm");
    io_save_mask_pbm(path, mask, h, w);
  });
}

int sige_load_mask_pbm(const char* path, uint8_t* mask, size_t cap, int* h, int* w) {
  return guarded([&] {
    need(path, "load_mask_pbm");
    need(h, "load_mask_pbm");
    need(w, "load_mask_pbm");
    io_load_mask_pbm(path, h, w, mask, cap);
  });
}

int sige_save_block_stack(const char* prefix, const float* host, int count, int channels, int block, int overlap,
                          int origin_block, int origin_h, int origin_w, const int32_t* idx) {
  return guarded([&] {
    need(prefix, "save_block_stack");
    if (count < 0 || channels < 0 || block < 1 || overlap < 0)
      throw ConfigError("save_block_stack: bad block stack geometry");
    if (count) {
      need(host, "save_block_stack");
      need(idx, "save_block_stack");
    }
    io_save_block_stack(prefix, host, count, channels, block, overlap, origin_block, origin_h, origin_w, idx);
  });
}

int sige_load_block_stack(const char* prefix, float* host, size_t cap, int32_t* idx, size_t idx_cap, int* meta) {
  return guarded([&] {
    need(prefix, "load_block_stack");
    need(meta, "load_block_stack");
    io_load_block_stack(prefix, meta, host, cap, idx, idx_cap);
  });
}

}  // extern "C"
