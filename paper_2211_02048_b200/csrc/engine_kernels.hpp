// engine_kernels.hpp — device-side descriptors and launchers of the engine
// (the production sparse_forward path). Activations inside the engine are
// NHWC fp32 ("channels-last"): a pixel's channels are one contiguous run, so
// gathers move whole 16-byte vectors and the tensor-core operand rows come out
// K-contiguous. External tensors (the edited input, the final output) are
// NCHW, the reference layout (proj/include/sige/tensor.hpp:12-39).
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.hpp"

namespace sige_b200 {

enum Layout : int { kNHWC = 0, kNCHW = 1 };

// An activation as a consumer sees it: the stored tensor (physical
// h >> up, w >> up), its layout, the pending element-wise chain (Flow::pending,
// graph.cpp:545-553) and the nearest-upsample shift folded into the index
// arithmetic instead of materialising upsample_nearest2x (tensor.cpp:69-83).
struct Src {
  const float* ptr = nullptr;
  int layout = kNHWC;
  int n = 1, c = 0, h = 0, w = 0;  // logical dims
  int up = 0;                       // log2 upsample factor
  int half = 0;                     // storage is fp16 (activation buffers), else fp32
  DevEpilogue epi;
  // fp16 channels-last copy of the same values (F16 mode): the tensor-core
  // conv streams it with cp.async when no element-wise chain is pending.
  const void* twin = nullptr;
  int twin_c = 0;  // channel stride of the twin (>= c, zero-padded; 0 = c)
  // GroupNorm folded from raw statistics (F16 dense-fallback ResBlocks): when
  // gn_stats != nullptr the chain is [scale-shift from (sum, sum of squares)
  // per (n, group) in doubles, then `epi`]; scale = gamma / sqrt(var + eps),
  // shift = beta - mean * scale (fold_stats, norm.cpp:66-90).
  const double* gn_stats = nullptr;
  int gn_groups = 0;
  float gn_eps = 0.0f;
  double gn_count = 0.0;  // values per (n, group)
  const float* gn_gamma = nullptr;
  const float* gn_beta = nullptr;
};

#ifdef __CUDACC__
// Raw stored value of logical pixel (n, ch, y, x) (caller bounds-checks).
__device__ __forceinline__ float src_raw(const Src& s, int n, int ch, int y, int x) {
  int ph = s.h >> s.up, pw = s.w >> s.up;
  int py = y >> s.up, px = x >> s.up;
  size_t off = s.layout == kNHWC ? ((static_cast<size_t>(n) * ph + py) * pw + px) * s.c + ch
                                 : ((static_cast<size_t>(n) * s.c + ch) * ph + py) * pw + px;
  if (s.half) return __half2float(reinterpret_cast<const __half*>(s.ptr)[off]);
  return __ldg(s.ptr + off);
}
__device__ __forceinline__ float src_val(const Src& s, int n, int ch, int y, int x) {
  return dev_epi(s.epi, src_raw(s, n, ch, y, x), ch, s.c, n);
}
#endif

// What a conv does with its (acc + bias) value at output pixel p.
enum OutMode : int {
  kStore = 0,        // dst[p] = v                      (scatter_inplace, kernels.cpp:88-106)
  kResMain = 1,      // dst[p] = v + aux[p]             (main tiles, kernels.cpp:306-318)
  kResShortcut = 2,  // dst[p] = dst[p] + (v - aux[p])  (shortcut tiles, kernels.cpp:320-334)
  kAddSrc = 3,       // dst[p] = v + addend(p)          (dense ResBlock join add(m, sc), graph.cpp:812)
};

// The tile list a conv runs over: `count` triplets {n, r, c} (output-res
// tile origins, BlockIndexSet order), count read from the device when
// count_dev != nullptr (produced by the on-device IndexPlan).
struct Tiles {
  const int32_t* idx = nullptr;
  const int32_t* count_dev = nullptr;
  int count = 0;     // used when count_dev == nullptr
  int capacity = 0;  // upper bound for grid sizing
  int bh = 0, bw = 0;  // tile shape at output resolution (square for sparse)
};

struct Dst {
  float* ptr = nullptr;  // NHWC, (n, h, w, c)
  int n = 1, c = 0, h = 0, w = 0;
  int mode = kStore;
  const float* aux = nullptr;  // NHWC, same shape (original shortcut)
  Src addend;                  // kAddSrc
  // Optional activation output: act[p] = act_epi(value written at p) — the
  // consumer's pending GroupNorm scale-shift + activation evaluated once per
  // output pixel (NHWC, same shape; fp16 when act_half).
  void* act = nullptr;
  int act_half = 0;
  DevEpilogue act_epi;
  // Identity-shortcut join fused into conv2 (kResMain, kernels.cpp:320-334):
  // main-tile pixels that also lie in an active shortcut tile get
  // + (x - aux); the shortcut-tile pixels outside every active main tile are
  // joined (dst += x - aux) by the same kernel's join phase. join_bm / main_bm:
  // activity bitmaps of the shortcut (join_b) and main (main_b) tile grids.
  const uint32_t* join_bm = nullptr;
  const uint32_t* main_bm = nullptr;
  int join_b = 0, main_b = 0;
  int join_bm_words = 0, main_bm_words = 0;  // words per sample (grouped requests), 0: one shared bitmap
  Src join_x;    // the block input x
  Tiles join_tiles;  // the shortcut tile list
  // Optional GroupNorm statistics of the written values: += (sum, sum of
  // squares) per (n, group) into gn_stats[2 * (n * gn_groups + g)] (doubles,
  // zeroed by the caller) — the next layer folds them (Src::gn_stats).
  double* gn_stats = nullptr;
  int gn_groups = 0;
  // Tensor-core conv only: skip the main (fp32) store — the value is consumed
  // through `act` alone (conv1 of a ResBlock whose conv2 stages act1); needs
  // c_out % 16 == 0 and c % 4 == 0 (the vector epilogue path).
  int no_main = 0;
};


// TMA descriptors of a packed weight tensor, one per N-slice width
// (16, 32, 64, 128, 256) with the taps batched per ring stage.
struct TcMaps {
  CUtensorMap m[5];
  int tps[5];
};

struct ConvW {
  int c_in = 0, c_out = 0, k = 1, stride = 1;
  const float* w = nullptr;     // (c_out, c_in, k, k) reference layout
  const float* bias = nullptr;  // c_out or nullptr
  const void* w_tc = nullptr;   // tcgen05 packing [chunk][tap][n_pad][128 B K row] (conv_tc.cu)
  size_t w_tc_bytes = 0;        // bytes of the packing
  int n_pad = 0;                // c_out rounded up for the tensor-core N dimension
  int k_pad = 0;                // channels rounded up per tap for the K dimension
  TcMaps maps{};
};

// Fused gather -> conv -> scatter over tiles (exact fp32 CUDA-core path:
// reference order, no FMA; bit-exact). conv_exact.cu.
void launch_conv_exact(const Src& src, const Tiles& tiles, const ConvW& cw, const Dst& dst,
                       int math, cudaStream_t st);
// Same contract on tcgen05 tensor cores (kind::tf32, fp32 TMEM accumulators).
// conv_tc.cu.
// gtl (optional): device stamp buffer of the engine's graph timeline — this
// launch records [first CTA start, last CTA end] at gtl[2 idx], gtl[2 idx + 1]
// and its first dependency-wait exit at gtl[2 kTimelineSlots + idx] (globaltimer).
constexpr int kTimelineSlots = 1024;
// pad >= 0 overrides the conv padding (k - 1) / 2 (op-level conv_on_blocks:
// the gathered window already carries the halo, kernels.cpp:391-421).
// Returns the launch's grid size (0: nothing launched).
int launch_conv_tc(const Src& src, const Tiles& tiles, const ConvW& cw, const Dst& dst, int f16,
                   cudaStream_t st, int sm_budget = 0, unsigned long long* gtl = nullptr, int gtl_idx = 0,
                   int pad = -1);
// Packs reference-layout weights for launch_conv_tc (fills w_tc, n_pad,
// k_pad and the TMA descriptors of `cw`).
// Developer instrumentation (SIGE_TC_GTL=1): per-launch conv spans, read + reset.
int debug_conv_timeline(unsigned long long* out, int cap);
// CTA 0's phase marks (64 globaltimer slots per launch, 0 = not reached).
int debug_conv_marks(unsigned long long* out, int cap);
void pack_weights_tc(const float* w_dev_ref, int c_out, int c_in, int k, int f16, ConvW* cw,
                     cudaStream_t st);

// On-device IndexPlan (graph.cpp:506-528): for every entry e, tile (r, c) of
// an (h_e, w_e, b_e) grid is active iff the full-resolution difference mask
// has a set pixel in the rectangle that dilate_full, resampling (max-pool
// down / replicate up) and dilate_scale map onto that tile. One CTA per entry
// writes the active tiles in row-major order, replicated n-major.
struct PlanEntryDev {
  int h, w, b;
  int32_t* idx;    // capacity triplets
  int32_t* count;  // device int
  int capacity;
  uint32_t* bm;    // activity bitmap of the (h/b, w/b) tile grid, row-major (one per sample when grouped)
};
// Both set *any = 1 when at least one pixel is set (the caller zeroes it).
// per_sample / masks > 1 (grouped requests): one mask, bit mask and any flag
// per sample (bits: masks x h x ceil(w/32) words).
void launch_mask_bits(const float* orig, const float* edited, int n, int c, int h, int w, float thr,
                      uint32_t* bits, uint8_t* mask_u8, int32_t* any, cudaStream_t st, int per_sample = 0);
void launch_mask_u8_to_bits(const uint8_t* mask, int h, int w, uint32_t* bits, int32_t* any,
                            cudaStream_t st, int masks = 1);
void launch_plan(const uint32_t* bits, int H, int W, int dilate_full, int dilate_scale, int batch,
                 const PlanEntryDev* entries_dev, int num_entries, cudaStream_t st, int per_sample = 0);

// GroupNorm statistics + fold (norm.cpp:25-90) over a full NHWC tensor,
// writing scale/shift (n*C). exact=1 follows the reference's sequential
// double accumulation order (bit-exact); 0 uses a parallel tree.
void launch_gn_fold(const Src& x, int groups, float eps, const float* gamma, const float* beta,
                    float* scale, float* shift, double* scratch, int scratch_len, int exact,
                    cudaStream_t st);
// Batch-kind fold of running statistics (graph.cpp:313-320).
void launch_bn_fold(int c, float eps, const float* gamma, const float* beta, const float* rmean,
                    const float* rvar, float* scale, float* shift, cudaStream_t st);

// dst (NHWC or NCHW per dst_layout, full tensor) = value of `src` at every
// pixel (pending chain + upsample applied): flush()/materialize().
void launch_materialize(const Src& src, float* dst, int dst_layout, cudaStream_t st);
// Final-tile copy: dst (NCHW) at tiles = epi(src) (apply_epilogue_on_blocks +
// scatter into the cached final output, graph.cpp:891-898).
void launch_tiles_apply(const Src& src, const Tiles& tiles, float* dst, int dst_layout,
                        cudaStream_t st);
// Identity-shortcut join at shortcut tiles: dst[p] = dst[p] + (src(p) - aux[p]).
void launch_identity_join(const Src& src, const Tiles& tiles, const Dst& dst, cudaStream_t st);
// Restore tiles of a working buffer from its cache entry (same layout).
struct RestoreJob {
  float* dst;
  const float* src;
  const int32_t* idx;
  const int32_t* count;
  int n, c, h, w, b, layout;
  int half;  // 2-byte elements (fp16 activation buffers)
};
// dst (NHWC, fp16 when half else fp32) = value of `src` (pending chain applied)
// at every pixel: the activation buffer a conv consumes instead of re-applying
// GroupNorm scale-shift + SiLU per staged window element.
void launch_materialize_act(const Src& src, void* dst, int half, cudaStream_t st);
void launch_restore(const RestoreJob* jobs_dev, int num_jobs, int max_tiles, cudaStream_t st);
// out (NCHW, full) = *any ? value of `result` : cached_final — the empty-mask
// short-circuit of sparse_forward (graph.cpp:665-668) folded into the final copy.
void launch_finalize(const Src& result, const float* cached_final, const int32_t* any, float* out,
                     cudaStream_t st, int per_sample = 0);
// Elementwise a + b over n values (dense ResBlock sum in precompute).
void launch_add(const float* a, const float* b, float* out, size_t n, cudaStream_t st);
// Same, also writing out_h16 = fp16(out) when out_h16 != nullptr.
void launch_add_h(const float* a, const float* b, float* out, void* out_h16, size_t n, cudaStream_t st);
// NCHW fp32 (n, c, h, w) -> NHWC fp16 with the channels zero-padded to c_pad
// (the fp16 twin of the edited input that the first convolution streams).
void launch_input_twin(const float* in, int n, int c, int h, int w, int c_pad, void* out, cudaStream_t st);
// dst_h16 = fp16(src) elementwise (same layout).
void launch_to_half(const float* src, void* dst_h16, size_t n, cudaStream_t st);
// Config 3 (SPADE): nearest resize NCHW -> NHWC (+ fp16 twin padded to c16
// channels; out or out16 may be null), and the SPADE modulation over tiles
// (tiles != nullptr) or every pixel.
void launch_resize_nhwc(const float* in, int n, int c, int H, int W, int h, int w, float* out, void* out16, int c16,
                        cudaStream_t st);
void launch_spade_mod(const Src& x, const float* sc, const float* sh, const float* gb, int act, const Tiles* tiles,
                      float* out, void* out16, cudaStream_t st);
// Layout conversions.
void launch_nchw_to_nhwc(const float* in, float* out, int n, int c, int h, int w, cudaStream_t st);
void launch_nhwc_to_nchw(const float* in, float* out, int n, int c, int h, int w, cudaStream_t st);

}  // namespace sige_b200
