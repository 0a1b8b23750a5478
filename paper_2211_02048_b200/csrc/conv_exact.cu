// conv_exact.cu — fused gather -> conv -> scatter on CUDA cores, in the
// reference's accumulation order (detail::conv2d_raw, proj/src/conv.cpp:33-79):
// per output acc = +0, then for ic, ky, kx: acc = acc + w*x with separately
// rounded multiply and add, bias added last. Zero-filled window cells stand in
// for skipped out-of-canvas taps; both give identical bits for finite inputs
// (test_kernels.cpp:306-351). This is the engine's bit-exact check mode
// (SIGE_MATH_EXACT) and its FP32-FMA mode; the fast path is conv_tc.cu.
//
// Work item = (tile, 32-output-channel chunk). The CTA stages the tile's input
// window 16 channels at a time in shared memory with the source's pending
// element-wise chain applied once per staged value (fused GroupNorm
// scale-shift + activation, graph.cpp:571-582), then each thread accumulates
// up to 16 output pixels of one output channel.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.hpp"
#include "engine_kernels.hpp"

namespace sige_b200 {

namespace {

constexpr int kCC = 16;     // staged input channels per chunk
constexpr int kOCC = 32;    // output channels per work item (one per lane)
constexpr int kThr = 128;   // 4 warps
constexpr int kMaxPix = 16; // output pixels per thread: bh*bw <= 4 * 16
constexpr int kWRow = kCC * 9 + 1;  // staged weights per output channel (+1: conflict-free lane rows)

__device__ __forceinline__ void write_out(const Dst& d, int n, int oc, int y, int x, float v) {
  const size_t p = ((static_cast<size_t>(n) * d.h + y) * d.w + x) * d.c + oc;
  switch (d.mode) {
    case kStore:
      d.ptr[p] = v;
      break;
    case kResMain:
      d.ptr[p] = __fadd_rn(v, d.aux[p]);
      break;
    case kResShortcut:
      d.ptr[p] = __fadd_rn(d.ptr[p], __fsub_rn(v, d.aux[p]));
      break;
    default:  // kAddSrc
      d.ptr[p] = __fadd_rn(v, src_val(d.addend, n, oc, y, x));
      break;
  }
}

template <int MATH>
__global__ void __launch_bounds__(kThr) k_conv_exact(Src src, Tiles t, ConvW cw, Dst dst) {
  extern __shared__ float win_s[];  // [win_h * win_w][kCC], channel fastest; then w_s[kOCC][kWRow]
  const int count = t.count_dev ? *t.count_dev : t.count;
  const int ci = cw.c_in, co = cw.c_out, k = cw.k, s = cw.stride, pad = (k - 1) / 2;
  const int win_h = (t.bh - 1) * s + k, win_w = (t.bw - 1) * s + k;
  const int npix = t.bh * t.bw;
  const int nocc = (co + kOCC - 1) / kOCC;
  const int lane = threadIdx.x & 31, pg = threadIdx.x >> 5;
  const int kk = k * k;
  float* w_s = win_s + win_h * win_w * kCC;
  for (int item = blockIdx.x; item < count * nocc; item += gridDim.x) {
    const int g = item / nocc, j = item % nocc;
    const int n = t.idx[3 * g], r0 = t.idx[3 * g + 1], c0 = t.idx[3 * g + 2];
    const int iy0 = r0 * s - pad, ix0 = c0 * s - pad;
    const int oc = j * kOCC + lane;
    const bool oc_ok = oc < co;
    float acc[kMaxPix];
#pragma unroll
    for (int i = 0; i < kMaxPix; ++i) acc[i] = 0.0f;
    for (int cb = 0; cb < ci; cb += kCC) {
      __syncthreads();
      const int nstage = win_h * win_w * kCC;
      for (int e = threadIdx.x; e < nstage; e += kThr) {
        const int cc = e % kCC, pix = e / kCC;
        const int ch = cb + cc, y = iy0 + pix / win_w, x = ix0 + pix % win_w;
        float v = 0.0f;
        if (ch < ci && y >= 0 && y < src.h && x >= 0 && x < src.w) v = src_val(src, n, ch, y, x);
        win_s[e] = v;
      }
      // the chunk's weights of the item's 32 output channels: one contiguous
      // run of cend * k * k floats per channel, read coalesced into shared memory
      // (per-lane global reads were 36-byte pieces 4.6 KB apart)
      const int cend = min(kCC, ci - cb);
      const int wrun = cend * kk;
      for (int e = threadIdx.x; e < kOCC * wrun; e += kThr) {
        const int row = e / wrun, col = e - row * wrun;
        const int ocr = j * kOCC + row;
        w_s[row * kWRow + col] = ocr < co ? __ldg(cw.w + (static_cast<size_t>(ocr) * ci + cb) * kk + col) : 0.0f;
      }
      __syncthreads();
      for (int cc = 0; cc < cend; ++cc) {
        float wk[9];
        const float* wp = w_s + lane * kWRow + cc * kk;
#pragma unroll
        for (int q = 0; q < 9; ++q) wk[q] = q < kk ? wp[q] : 0.0f;
#pragma unroll
        for (int i = 0; i < kMaxPix; ++i) {
          const int p = pg + 4 * i;
          if (p >= npix) break;
          const int py = p / t.bw, px = p % t.bw;
          const float* wrow = win_s + ((py * s) * win_w + px * s) * kCC + cc;
          float a = acc[i];
          for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) {
              const float xv = wrow[(ky * win_w + kx) * kCC];
              const float wv = wk[ky * k + kx];
              a = MATH == SIGE_MATH_FP32_FMA ? __fmaf_rn(wv, xv, a) : __fadd_rn(a, __fmul_rn(wv, xv));
            }
          acc[i] = a;
        }
      }
    }
    if (oc_ok) {
      const float b = cw.bias ? __ldg(cw.bias + oc) : 0.0f;
#pragma unroll
      for (int i = 0; i < kMaxPix; ++i) {
        const int p = pg + 4 * i;
        if (p >= npix) break;
        const int y = r0 + p / t.bw, x = c0 + p % t.bw;
        if (y >= dst.h || x >= dst.w) continue;
        write_out(dst, n, oc, y, x, cw.bias ? __fadd_rn(acc[i], b) : acc[i]);
      }
    }
  }
}

}  // namespace

void launch_conv_exact(const Src& src, const Tiles& tiles, const ConvW& cw, const Dst& dst,
                       int math, cudaStream_t st) {
  if (tiles.bh * tiles.bw > 4 * kMaxPix)
    throw ConfigError("conv (exact): tile of " + std::to_string(tiles.bh) + "x" +
                      std::to_string(tiles.bw) + " exceeds 64 output pixels");
  if (tiles.capacity == 0) return;
  const int win_h = (tiles.bh - 1) * cw.stride + cw.k, win_w = (tiles.bw - 1) * cw.stride + cw.k;
  const size_t smem = sizeof(float) * (win_h * win_w * kCC + kOCC * kWRow);
  const int nocc = (cw.c_out + kOCC - 1) / kOCC;
  const long long work = static_cast<long long>(tiles.capacity) * nocc;
  const int grid = static_cast<int>(std::max(1LL, std::min<long long>(work, sm_count() * 8LL)));
  if (math == SIGE_MATH_FP32_FMA)
    k_conv_exact<SIGE_MATH_FP32_FMA><<<grid, kThr, smem, st>>>(src, tiles, cw, dst);
  else
    k_conv_exact<SIGE_MATH_EXACT><<<grid, kThr, smem, st>>>(src, tiles, cw, dst);
  after_launch("k_conv_exact");
}

}  // namespace sige_b200
