// engine_kernels.cu — the engine's HBM-bound kernels: difference mask to a
// bit mask, the on-device IndexPlan (deterministic tile compaction), GroupNorm
// statistics, final-tile application, restores and layout conversions.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "common.hpp"
#include "engine_kernels.hpp"

namespace sige_b200 {

namespace {

inline int grid_cap(long long n, int threads) {
  long long g = (n + threads - 1) / threads;
  long long cap = static_cast<long long>(sm_count()) * 16;
  return static_cast<int>(std::max(1LL, std::min(g, cap)));
}

// ------------------------------------------------------ difference mask --
// compute_difference_mask (mask.cpp:14-32) straight into a row-major bit mask
// (ceil(W/32) words per row). grid.y splits the N*C planes; set bits are
// merged with atomicOr, so the result is order-independent.
// Grouped requests (per-sample masks): grid.z = sample, each with its own
// planes, bit mask (h x wpr words) and any flag.
__global__ void k_mask_bits(const float* __restrict__ o, const float* __restrict__ e, int planes,
                            int ppy, int h, int w, float thr, uint32_t* __restrict__ bits,
                            uint8_t* __restrict__ mask_u8, int32_t* __restrict__ any) {
  const long long hw = static_cast<long long>(h) * w;
  const int wpr = (w + 31) >> 5;
  o += static_cast<long long>(blockIdx.z) * planes * hw;
  e += static_cast<long long>(blockIdx.z) * planes * hw;
  bits += static_cast<long long>(blockIdx.z) * h * wpr;
  any += blockIdx.z;
  if (mask_u8) mask_u8 += blockIdx.z * hw;
  const int p0 = blockIdx.y * ppy, p1 = min(planes, p0 + ppy);
  // (the edited input is the caller's tensor: vector loads only when aligned)
  const bool vec = (w & 3) == 0 && ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(e)) & 15) == 0;
  const long long nq = vec ? hw >> 2 : hw;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nq;
       q += (long long)gridDim.x * blockDim.x) {
    uint32_t set = 0;  // bit j: pixel (vec ? 4q + j : q)
    if (vec) {
      for (int p = p0; p < p1; ++p) {
        float4 a = __ldg(reinterpret_cast<const float4*>(o + p * hw) + q);
        float4 b = __ldg(reinterpret_cast<const float4*>(e + p * hw) + q);
        set |= (fabsf(__fsub_rn(b.x, a.x)) > thr ? 1u : 0u) | (fabsf(__fsub_rn(b.y, a.y)) > thr ? 2u : 0u) |
               (fabsf(__fsub_rn(b.z, a.z)) > thr ? 4u : 0u) | (fabsf(__fsub_rn(b.w, a.w)) > thr ? 8u : 0u);
        if (set == 15u) break;
      }
    } else {
      for (int p = p0; p < p1 && !set; ++p)
        set = fabsf(__fsub_rn(__ldg(e + p * hw + q), __ldg(o + p * hw + q))) > thr ? 1u : 0u;
    }
    if (!set) continue;
    *any = 1;
    long long pix = vec ? (q << 2) : q;
    int y = static_cast<int>(pix / w), x = static_cast<int>(pix % w);
    for (int j = 0; j < (vec ? 4 : 1); ++j) {
      if (!(set >> j & 1u)) continue;
      atomicOr(bits + static_cast<long long>(y) * wpr + ((x + j) >> 5), 1u << ((x + j) & 31));
      if (mask_u8) mask_u8[pix + j] = 1;
    }
  }
}

__global__ void k_mask_u8_to_bits(const uint8_t* __restrict__ m, int h, int w, uint32_t* bits,
                                  int32_t* __restrict__ any) {
  const int wpr = (w + 31) >> 5;
  m += static_cast<long long>(blockIdx.z) * h * w;  // grouped: one mask per sample
  bits += static_cast<long long>(blockIdx.z) * h * wpr;
  any += blockIdx.z;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)h * wpr;
       q += (long long)gridDim.x * blockDim.x) {
    int y = static_cast<int>(q / wpr), wd = static_cast<int>(q % wpr);
    uint32_t v = 0;
    for (int j = 0; j < 32; ++j) {
      int x = wd * 32 + j;
      if (x < w && m[static_cast<long long>(y) * w + x]) v |= 1u << j;
    }
    bits[q] = v;
    if (v) *any = 1;
  }
}

// -------------------------------------------------------------- plan ----
__device__ __forceinline__ bool rect_any(const uint32_t* bits, int wpr, int y0, int y1, int x0,
                                         int x1) {
  int wa = x0 >> 5, wb = x1 >> 5;
  uint32_t ma = 0xffffffffu << (x0 & 31);
  uint32_t mb = 0xffffffffu >> (31 - (x1 & 31));
  for (int y = y0; y <= y1; ++y) {
    const uint32_t* row = bits + static_cast<long long>(y) * wpr;
    if (wa == wb) {
      if (row[wa] & ma & mb) return true;
    } else {
      if (row[wa] & ma) return true;
      for (int k = wa + 1; k < wb; ++k)
        if (row[k]) return true;
      if (row[wb] & mb) return true;
    }
  }
  return false;
}

// One CTA per plan entry. The rectangle for tile (R, C): its clipped pixels
// dilated by dilate_scale at the entry resolution, mapped to full resolution
// (max-pool down: factor f rows per cell; replicate up: y/u), dilated by
// dilate_full, clipped — composition of dilate_mask (mask.cpp:55-80),
// downsample_mask (mask.cpp:34-53) / replicate_mask (graph.cpp:485-500) and
// the "any pixel in tile" test of mask_to_block_indices (mask.cpp:113-127).
// per_sample (grouped requests): one pass per sample over its own bit mask,
// tiles appended n-major ((n, r, c) order) and one activity bitmap per sample;
// otherwise one pass over the shared mask, replicated for every sample
// (mask_to_block_indices, mask.cpp:129-134).
__global__ void k_plan(const uint32_t* __restrict__ gbits_all, int H, int W, int df, int ds, int batch,
                       const PlanEntryDev* __restrict__ entries, int use_smem, int per_sample) {
  extern __shared__ uint32_t sbits[];
  __shared__ int warp_sums[32];
  __shared__ int base;
  const int wpr = (W + 31) >> 5;
  const PlanEntryDev e = entries[blockIdx.x];
  if (threadIdx.x == 0) base = 0;
  const int passes = per_sample ? batch : 1;
  for (int pass = 0; pass < passes; ++pass) {
  const uint32_t* gbits = gbits_all + static_cast<long long>(pass) * H * wpr;
  const uint32_t* bits = gbits;
  __syncthreads();  // previous pass done with the shared bits
  if (use_smem) {
    for (int i = threadIdx.x; i < H * wpr; i += blockDim.x) sbits[i] = gbits[i];
    bits = sbits;
  }
  const int h = e.h, w = e.w, b = e.b;
  const int ty = (h + b - 1) / b, tx = (w + b - 1) / b, tiles = ty * tx;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool down_y = h <= H, down_x = w <= W;
  // The tile rectangle is separable (rows from the tile row, columns from the
  // tile column): OR each tile row's full-resolution row range into one
  // bit row first, so a tile tests 1-2 words instead of scanning ~20-40 rows
  // (almost every tile of a small edit is inactive, the worst case of the scan).
  uint32_t* rowor = sbits + H * wpr;
  const bool sep = use_smem && ty * wpr <= 2 * H * wpr;
  if (sep) {
    for (int k = threadIdx.x; k < ty * wpr; k += blockDim.x) {
      const int r = k / wpr, wd = k - r * wpr, R = r * b;
      const int ly0 = max(0, R - ds), ly1 = min(h - 1, min(h, R + b) - 1 + ds);
      int fy0, fy1;
      if (down_y) {
        const int f = H / h;
        fy0 = ly0 * f;
        fy1 = ly1 * f + f - 1;
      } else {
        const int u = h / H;
        fy0 = ly0 / u;
        fy1 = ly1 / u;
      }
      fy0 = max(0, fy0 - df);
      fy1 = min(H - 1, fy1 + df);
      uint32_t acc = 0;
      for (int y = fy0; y <= fy1; ++y) acc |= bits[y * wpr + wd];
      rowor[k] = acc;
    }
  }
  __syncthreads();
  uint32_t* bm = e.bm ? e.bm + static_cast<long long>(pass) * ((tiles + 31) >> 5) : nullptr;
  for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
    const int t = t0 + threadIdx.x;
    bool on = false;
    int R = 0, Cc = 0;
    if (t < tiles) {
      R = (t / tx) * b;
      Cc = (t % tx) * b;
      int ly0 = max(0, R - ds), ly1 = min(h - 1, min(h, R + b) - 1 + ds);
      int lx0 = max(0, Cc - ds), lx1 = min(w - 1, min(w, Cc + b) - 1 + ds);
      int fy0, fy1, fx0, fx1;
      if (down_y) {
        int f = H / h;
        fy0 = ly0 * f;
        fy1 = ly1 * f + f - 1;
      } else {
        int u = h / H;
        fy0 = ly0 / u;
        fy1 = ly1 / u;
      }
      if (down_x) {
        int f = W / w;
        fx0 = lx0 * f;
        fx1 = lx1 * f + f - 1;
      } else {
        int u = w / W;
        fx0 = lx0 / u;
        fx1 = lx1 / u;
      }
      fy0 = max(0, fy0 - df);
      fy1 = min(H - 1, fy1 + df);
      fx0 = max(0, fx0 - df);
      fx1 = min(W - 1, fx1 + df);
      on = sep ? rect_any(rowor + (t / tx) * wpr, wpr, 0, 0, fx0, fx1) : rect_any(bits, wpr, fy0, fy1, fx0, fx1);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) warp_sums[wid] = __popc(bal);
    if (bm && lane == 0 && t0 + wid * 32 < tiles) bm[(t0 + wid * 32) >> 5] = bal;  // tile activity bitmap
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
      }
      if (lane < nw) warp_sums[lane] = v;
    }
    __syncthreads();
    const int slot = base + (wid ? warp_sums[wid - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
    if (on && slot < e.capacity) {
      e.idx[3 * slot] = pass;
      e.idx[3 * slot + 1] = R;
      e.idx[3 * slot + 2] = Cc;
    }
    const int chunk_total = warp_sums[nw - 1];
    __syncthreads();
    if (threadIdx.x == 0) base += chunk_total;
    __syncthreads();
  }
  }  // passes
  if (per_sample) {
    if (threadIdx.x == 0) *e.count = min(base, e.capacity);
    return;
  }
  const int per = base;
  for (int n = 1; n < batch; ++n)
    for (int i = threadIdx.x; i < per; i += blockDim.x) {
      const int d = n * per + i;
      if (d < e.capacity) {
        e.idx[3 * d] = n;
        e.idx[3 * d + 1] = e.idx[3 * i + 1];
        e.idx[3 * d + 2] = e.idx[3 * i + 2];
      }
    }
  if (threadIdx.x == 0) *e.count = min(per * batch, e.capacity);
}

// ------------------------------------------------------------ GroupNorm --
// compute_norm_stats + fold_stats (norm.cpp:25-90). Exact: one thread per
// (n, group) with the reference's sequential double sums (channel in group,
// rows, columns), so mean/var round identically.
__global__ void k_gn_exact(Src x, int groups, float eps, const float* __restrict__ gamma,
                           const float* __restrict__ beta, float* __restrict__ scale,
                           float* __restrict__ shift) {
  const int cpg = x.c / groups;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < x.n * groups; q += gridDim.x * blockDim.x) {
    const int n = q / groups, g = q % groups;
    const double count = static_cast<double>(cpg) * x.h * x.w;
    double sum = 0.0;
    for (int ic = g * cpg; ic < (g + 1) * cpg; ++ic)
      for (int y = 0; y < x.h; ++y)
        for (int xx = 0; xx < x.w; ++xx) sum = __dadd_rn(sum, static_cast<double>(src_val(x, n, ic, y, xx)));
    const double mean = __ddiv_rn(sum, count);
    double sq = 0.0;
    for (int ic = g * cpg; ic < (g + 1) * cpg; ++ic)
      for (int y = 0; y < x.h; ++y)
        for (int xx = 0; xx < x.w; ++xx) {
          double d = __dadd_rn(static_cast<double>(src_val(x, n, ic, y, xx)), -mean);
          sq = __dadd_rn(sq, __dmul_rn(d, d));
        }
    const float fmean = __double2float_rn(mean), fvar = __double2float_rn(__ddiv_rn(sq, count));
    for (int ic = g * cpg; ic < (g + 1) * cpg; ++ic) {
      const float s = __fdiv_rn(gamma[ic], __fsqrt_rn(__fadd_rn(fvar, eps)));
      scale[n * x.c + ic] = s;
      shift[n * x.c + ic] = __fsub_rn(beta[ic], __fmul_rn(fmean, s));
    }
  }
}

// Parallel tree version: CTA per (n, group), double partial sums.
__global__ void k_gn_fast(Src x, int groups, float eps, const float* __restrict__ gamma,
                          const float* __restrict__ beta, float* __restrict__ scale,
                          float* __restrict__ shift) {
  __shared__ double red[32];
  __shared__ double s_mean;
  const int n = blockIdx.x / groups, g = blockIdx.x % groups;
  const int cpg = x.c / groups;
  const long long per = static_cast<long long>(cpg) * x.h * x.w;
  const double count = static_cast<double>(per);
  auto reduce = [&](double v) -> double {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x < 32) {
      t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    __syncthreads();
    return t;
  };
  // element q of the group: channel-fastest for NHWC coalescing
  double s = 0.0;
  for (long long q = threadIdx.x; q < per; q += blockDim.x) {
    int ic = g * cpg + static_cast<int>(q % cpg);
    long long pix = q / cpg;
    s += static_cast<double>(src_val(x, n, ic, static_cast<int>(pix / x.w), static_cast<int>(pix % x.w)));
  }
  s = reduce(s);
  if (threadIdx.x == 0) s_mean = s / count;
  __syncthreads();
  const double mean = s_mean;
  double sq = 0.0;
  for (long long q = threadIdx.x; q < per; q += blockDim.x) {
    int ic = g * cpg + static_cast<int>(q % cpg);
    long long pix = q / cpg;
    double d = static_cast<double>(src_val(x, n, ic, static_cast<int>(pix / x.w), static_cast<int>(pix % x.w))) - mean;
    sq += d * d;
  }
  sq = reduce(sq);
  if (threadIdx.x < cpg) {
    const int ic = g * cpg + threadIdx.x;
    const float fmean = static_cast<float>(mean), fvar = static_cast<float>(sq / count);
    const float sc = __fdiv_rn(gamma[ic], __fsqrt_rn(__fadd_rn(fvar, eps)));
    scale[n * x.c + ic] = sc;
    shift[n * x.c + ic] = __fsub_rn(beta[ic], __fmul_rn(fmean, sc));
  }
}

// Multi-CTA statistics for the tensor-core mode: CTA (n, s) owns pixel range s
// of sample n, one thread per channel (NHWC rows are read coalesced),
// per-thread double sum / sum of squares in pixel order, then a fixed-order
// reduction over the group's channels -> partial[(n*groups + g)*S + s].
// Deterministic (fixed partition and order) but not the reference's rounding.
__global__ void k_gn_partial(Src x, int groups, int S, double* __restrict__ part) {
  const int n = blockIdx.x / S, s = blockIdx.x % S;
  const long long hw = static_cast<long long>(x.h) * x.w;
  const long long p0 = hw * s / S, p1 = hw * (s + 1) / S;
  extern __shared__ double red[];  // [2][C]
  for (int c = threadIdx.x; c < x.c; c += blockDim.x) {
    double a = 0.0, q = 0.0;
    for (long long p = p0; p < p1; ++p) {
      const double v = static_cast<double>(src_val(x, n, c, static_cast<int>(p / x.w), static_cast<int>(p % x.w)));
      a += v;
      q += v * v;
    }
    red[c] = a;
    red[x.c + c] = q;
  }
  __syncthreads();
  const int cpg = x.c / groups;
  for (int g = threadIdx.x; g < groups; g += blockDim.x) {
    double a = 0.0, q = 0.0;
    for (int c = g * cpg; c < (g + 1) * cpg; ++c) {
      a += red[c];
      q += red[x.c + c];
    }
    part[(2 * (static_cast<long long>(n) * groups + g)) * S + s] = a;
    part[(2 * (static_cast<long long>(n) * groups + g) + 1) * S + s] = q;
  }
}

__global__ void k_gn_final(int n_groups_total, int groups, int S, int C, long long count_per_group,
                           float eps, const double* __restrict__ part, const float* __restrict__ gamma,
                           const float* __restrict__ beta, float* __restrict__ scale, float* __restrict__ shift) {
  const int cpg = C / groups;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_groups_total * cpg; q += gridDim.x * blockDim.x) {
    const int ng = q / cpg, ci = q % cpg;
    const int n = ng / groups, g = ng % groups;
    double a = 0.0, sq = 0.0;
    for (int s = 0; s < S; ++s) {
      a += part[(2LL * ng) * S + s];
      sq += part[(2LL * ng + 1) * S + s];
    }
    const double cnt = static_cast<double>(count_per_group);
    const double mean = a / cnt;
    double var = sq / cnt - mean * mean;
    if (var < 0.0) var = 0.0;
    const int c = g * cpg + ci;
    const float sc = __fdiv_rn(gamma[c], __fsqrt_rn(__fadd_rn(static_cast<float>(var), eps)));
    scale[n * C + c] = sc;
    shift[n * C + c] = __fsub_rn(beta[c], __fmul_rn(static_cast<float>(mean), sc));
  }
}

__global__ void k_bn_fold(int c, float eps, const float* gamma, const float* beta, const float* rm,
                          const float* rv, float* scale, float* shift) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x) {
    const float s = __fdiv_rn(gamma[i], __fsqrt_rn(__fadd_rn(rv[i], eps)));
    scale[i] = s;
    shift[i] = __fsub_rn(beta[i], __fmul_rn(rm[i], s));
  }
}

// ------------------------------------------------------- elementwise ----
__global__ void k_materialize(Src s, float* __restrict__ dst, int dst_layout) {
  const long long total = static_cast<long long>(s.n) * s.c * s.h * s.w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int n, ch, y, x;
    if (dst_layout == kNHWC) {
      ch = static_cast<int>(q % s.c);
      long long p = q / s.c;
      x = static_cast<int>(p % s.w);
      p /= s.w;
      y = static_cast<int>(p % s.h);
      n = static_cast<int>(p / s.h);
    } else {
      x = static_cast<int>(q % s.w);
      long long p = q / s.w;
      y = static_cast<int>(p % s.h);
      p /= s.h;
      ch = static_cast<int>(p % s.c);
      n = static_cast<int>(p / s.c);
    }
    dst[q] = src_val(s, n, ch, y, x);
  }
}

// Per tile element helper: maps a flat index over (tile, pixel, channel) with
// channel fastest; returns false when the tile is inactive or the pixel is
// outside the canvas (fringe clipping, kernels.cpp:93-95).
__device__ __forceinline__ bool tile_elem(const Tiles& t, int count, int c, int h, int w,
                                          long long q, int& n, int& y, int& x, int& ch) {
  const long long per = static_cast<long long>(t.bh) * t.bw * c;
  const long long g = q / per;
  if (g >= count) return false;
  int rem = static_cast<int>(q - g * per);
  ch = rem % c;
  int cell = rem / c;
  n = t.idx[3 * g];
  y = t.idx[3 * g + 1] + cell / t.bw;
  x = t.idx[3 * g + 2] + cell % t.bw;
  return y < h && x < w;
}

// Programmatic dependent launch for the small kernels between convolutions:
// wait for the previous grid (everything read here was produced by it or
// earlier), then let the next kernel launch and run its own prologue.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__global__ void k_tiles_apply(Src s, Tiles t, float* __restrict__ dst, int dst_layout) {
  pdl_enter();
  const int count = t.count_dev ? *t.count_dev : t.count;
  const long long total = static_cast<long long>(count) * t.bh * t.bw * s.c;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int n, y, x, ch;
    if (!tile_elem(t, count, s.c, s.h, s.w, q, n, y, x, ch)) continue;
    size_t off = dst_layout == kNHWC ? ((static_cast<size_t>(n) * s.h + y) * s.w + x) * s.c + ch
                                     : ((static_cast<size_t>(n) * s.c + ch) * s.h + y) * s.w + x;
    dst[off] = src_val(s, n, ch, y, x);
  }
}

__global__ void k_identity_join(Src s, Tiles t, Dst d) {
  pdl_enter();
  const int count = t.count_dev ? *t.count_dev : t.count;
  const long long total = static_cast<long long>(count) * t.bh * t.bw * d.c;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int n, y, x, ch;
    if (!tile_elem(t, count, d.c, d.h, d.w, q, n, y, x, ch)) continue;
    const size_t p = ((static_cast<size_t>(n) * d.h + y) * d.w + x) * d.c + ch;
    const float v = __fadd_rn(d.ptr[p], __fsub_rn(src_val(s, n, ch, y, x), d.aux[p]));
    d.ptr[p] = v;
    if (d.act && d.act_half) static_cast<__half*>(d.act)[p] = __float2half_rn(v);  // fp16 twin
  }
}

__global__ void k_restore(const RestoreJob* __restrict__ jobs, int max_tiles) {
  pdl_enter();
  const RestoreJob j = jobs[blockIdx.y];
  const int count = min(*j.count, max_tiles);
  const int esz = j.half ? 2 : 4;
  if (j.layout == kNHWC && (j.c * esz) % 16 == 0) {
    // Channels-last: each clipped tile row is one contiguous run of
    // (cells x C) elements — copied as 16-byte vectors, one tile per CTA pass.
    const int vrow_full = j.b * j.c * esz / 16;
    for (int g = blockIdx.x; g < count; g += gridDim.x) {
      const int n = j.idx[3 * g], y0 = j.idx[3 * g + 1], x0 = j.idx[3 * g + 2];
      const int rows = min(j.b, j.h - y0), cells = min(j.b, j.w - x0);
      const int vrow = cells * j.c * esz / 16;
      // 4 vectors in flight per thread (one dependent load->store per pass
      // left the restore latency-bound)
      constexpr int kR = 4;
      for (int q0 = threadIdx.x; q0 < rows * vrow_full; q0 += blockDim.x * kR) {
        uint4 val[kR];
        size_t off[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
          const int q = q0 + u * blockDim.x;
          const int r = q / vrow_full, v = q - r * vrow_full;
          off[u] = ~size_t(0);
          if (q < rows * vrow_full && v < vrow) {
            off[u] = (((static_cast<size_t>(n) * j.h + y0 + r) * j.w + x0) * j.c) * esz / 16 + v;
            val[u] = reinterpret_cast<const uint4*>(j.src)[off[u]];
          }
        }
#pragma unroll
        for (int u = 0; u < kR; ++u)
          if (off[u] != ~size_t(0)) reinterpret_cast<uint4*>(j.dst)[off[u]] = val[u];
      }
    }
    return;
  }
  const long long per = static_cast<long long>(j.b) * j.b * j.c;
  const long long total = static_cast<long long>(count) * per;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const long long g = q / per;
    int rem = static_cast<int>(q - g * per);
    int ch, cell;
    if (j.layout == kNHWC) {
      ch = rem % j.c;
      cell = rem / j.c;
    } else {
      cell = rem % (j.b * j.b);
      ch = rem / (j.b * j.b);
    }
    const int n = j.idx[3 * g], y = j.idx[3 * g + 1] + cell / j.b, x = j.idx[3 * g + 2] + cell % j.b;
    if (y >= j.h || x >= j.w) continue;
    const size_t off = j.layout == kNHWC ? ((static_cast<size_t>(n) * j.h + y) * j.w + x) * j.c + ch
                                         : ((static_cast<size_t>(n) * j.c + ch) * j.h + y) * j.w + x;
    if (j.half)
      reinterpret_cast<__half*>(j.dst)[off] = reinterpret_cast<const __half*>(j.src)[off];
    else
      j.dst[off] = j.src[off];
  }
}

__global__ void k_materialize_act(Src s, void* __restrict__ dst, int half) {
  const long long total = static_cast<long long>(s.n) * s.c * s.h * s.w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int ch = static_cast<int>(q % s.c);
    long long p = q / s.c;
    const int x = static_cast<int>(p % s.w);
    p /= s.w;
    const int y = static_cast<int>(p % s.h);
    const int n = static_cast<int>(p / s.h);
    const float v = src_val(s, n, ch, y, x);
    if (half)
      static_cast<__half*>(dst)[q] = __float2half_rn(v);
    else
      static_cast<float*>(dst)[q] = v;
  }
}

__global__ void k_finalize(Src r, const float* __restrict__ cached, const int32_t* __restrict__ any,
                           float* __restrict__ out, int per_sample) {
  pdl_enter();
  const long long total = static_cast<long long>(r.n) * r.c * r.h * r.w;
  const long long per_n = static_cast<long long>(r.c) * r.h * r.w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const bool use = any[per_sample ? q / per_n : 0] != 0;  // empty mask -> cached final (graph.cpp:665-668)
    if (!use) {
      out[q] = cached[q];
      continue;
    }
    const int x = static_cast<int>(q % r.w);
    long long p = q / r.w;
    const int y = static_cast<int>(p % r.h);
    p /= r.h;
    out[q] = src_val(r, static_cast<int>(p / r.c), static_cast<int>(p % r.c), y, x);
  }
}

__global__ void k_add(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ o,
                      __half* __restrict__ oh, long long n) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const float v = __fadd_rn(a[q], b[q]);
    o[q] = v;
    if (oh) oh[q] = __float2half_rn(v);
  }
}

__global__ void k_input_twin(const float* __restrict__ in, int n, int c, int h, int w, int c_pad,
                             __half* __restrict__ out) {
  pdl_enter();
  const long long total = static_cast<long long>(n) * h * w * c_pad;
  const long long hw = static_cast<long long>(h) * w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int ch = static_cast<int>(q % c_pad);
    const long long p = q / c_pad;  // (n, pixel)
    const long long nn = p / hw, pix = p - nn * hw;
    out[q] = ch < c ? __float2half_rn(__ldg(in + (nn * c + ch) * hw + pix)) : __float2half_rn(0.0f);
  }
}

__global__ void k_to_half(const float* __restrict__ a, __half* __restrict__ o, long long n) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    o[q] = __float2half_rn(a[q]);
}

__global__ void k_nchw_to_nhwc(const float* __restrict__ in, float* __restrict__ out, int n, int c,
                               int h, int w) {
  const long long total = static_cast<long long>(n) * c * h * w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int ch = static_cast<int>(q % c);
    long long p = q / c;  // (n, y, x)
    long long hw = static_cast<long long>(h) * w;
    long long nn = p / hw, pix = p % hw;
    out[q] = in[(nn * c + ch) * hw + pix];
  }
}

__global__ void k_nhwc_to_nchw(const float* __restrict__ in, float* __restrict__ out, int n, int c,
                               int h, int w) {
  const long long total = static_cast<long long>(n) * c * h * w;
  const long long hw = static_cast<long long>(h) * w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long pix = q % hw;
    long long p = q / hw;
    int ch = static_cast<int>(p % c);
    long long nn = p / c;
    out[q] = in[(nn * hw + pix) * c + ch];
  }
}

// --------------------------------------------------------- SPADE (config 3) --
// Nearest resize of an NCHW map by integer factors into NHWC (+ an fp16 twin
// with channels padded to c16): the segmentation map at a block's resolution,
// and the RESIZE layer. down: (y f, x f); up: (y / u, x / u) — resize_nearest.
__global__ void k_resize_nhwc(const float* __restrict__ in, int n, int c, int H, int W, int h, int w,
                              float* __restrict__ out, __half* __restrict__ out16, int c16) {
  pdl_enter();
  const long long total = static_cast<long long>(n) * h * w * c16;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int ch = static_cast<int>(q % c16);
    long long p = q / c16;
    const int x = static_cast<int>(p % w);
    p /= w;
    const int y = static_cast<int>(p % h);
    const int in_n = static_cast<int>(p / h);
    const int sy = h <= H ? y * (H / h) : y / (h / H), sx = w <= W ? x * (W / w) : x / (w / W);
    const float v = ch < c ? __ldg(in + ((static_cast<size_t>(in_n) * c + ch) * H + sy) * W + sx) : 0.0f;
    const size_t pix = (static_cast<size_t>(in_n) * h + y) * w + x;
    if (ch < c && out) out[pix * c + ch] = v;
    if (out16) out16[pix * c16 + ch] = __float2half_rn(v);
  }
}

// SPADE modulation (Park et al. 2019): out = act((x sc + sh) (1 + gamma) + beta)
// with the folded param-free instance norm (sc, sh per sample and channel),
// gamma / beta the two halves of gb (NHWC, 2C channels), every operation
// rounded on its own (the restatement's order, oracle/spade.py). Over the
// tiles of `t` (sparse) or every pixel (t.idx == nullptr); NHWC fp32 out plus
// the fp16 twin the consuming conv streams.
__global__ void k_spade_mod(Src x, const float* __restrict__ sc, const float* __restrict__ sh,
                            const float* __restrict__ gb, int act, Tiles t, float* __restrict__ out,
                            __half* __restrict__ out16) {
  pdl_enter();
  const int c = x.c;
  const bool dense = t.idx == nullptr;
  const int count = dense ? 0 : (t.count_dev ? *t.count_dev : t.count);
  const long long total =
      dense ? static_cast<long long>(x.n) * x.h * x.w * c : static_cast<long long>(count) * t.bh * t.bw * c;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int n, y, xx, ch;
    if (dense) {
      ch = static_cast<int>(q % c);
      long long p = q / c;
      xx = static_cast<int>(p % x.w);
      p /= x.w;
      y = static_cast<int>(p % x.h);
      n = static_cast<int>(p / x.h);
    } else if (!tile_elem(t, count, c, x.h, x.w, q, n, y, xx, ch)) {
      continue;
    }
    const size_t pix = (static_cast<size_t>(n) * x.h + y) * x.w + xx;
    const int k = n * c + ch;
    const float v = src_val(x, n, ch, y, xx);
    const float nv = __fadd_rn(__fmul_rn(v, __ldg(sc + k)), __ldg(sh + k));
    const float g = __ldg(gb + pix * 2 * c + ch), b = __ldg(gb + pix * 2 * c + c + ch);
    float m = __fadd_rn(__fmul_rn(nv, __fadd_rn(1.0f, g)), b);
    if (act == SIGE_ACT_LEAKY_RELU) m = m > 0.0f ? m : __fmul_rn(0.2f, m);
    else if (act == SIGE_ACT_RELU) m = m > 0.0f ? m : 0.0f;
    out[pix * c + ch] = m;
    if (out16) out16[pix * c + ch] = __float2half_rn(m);
  }
}

}  // namespace

void launch_mask_bits(const float* orig, const float* edited, int n, int c, int h, int w, float thr,
                      uint32_t* bits, uint8_t* mask_u8, int32_t* any, cudaStream_t st, int per_sample) {
  const int wpr = (w + 31) >> 5;
  const int masks = per_sample ? n : 1;
  SIGE_CUDA(cudaMemsetAsync(bits, 0, sizeof(uint32_t) * h * wpr * masks, st));
  if (mask_u8) SIGE_CUDA(cudaMemsetAsync(mask_u8, 0, static_cast<size_t>(h) * w * masks, st));
  const long long hw = static_cast<long long>(h) * w;
  const long long nq = (w & 3) == 0 ? hw / 4 : hw;  // (grid sizing only: the kernel may fall back to scalar)
  const int planes = per_sample ? c : n * c;
  const int gx = static_cast<int>(std::min<long long>((nq + 255) / 256, 4096));
  int gy = std::min(planes, std::max(1, sm_count() * 8 / (gx * masks)));
  const int ppy = (planes + gy - 1) / gy;
  gy = (planes + ppy - 1) / ppy;
  k_mask_bits<<<dim3(gx, gy, masks), 256, 0, st>>>(orig, edited, planes, ppy, h, w, thr, bits, mask_u8, any);
  after_launch("k_mask_bits");
}

void launch_mask_u8_to_bits(const uint8_t* mask, int h, int w, uint32_t* bits, int32_t* any,
                            cudaStream_t st, int masks) {
  const int wpr = (w + 31) >> 5;
  k_mask_u8_to_bits<<<dim3(grid_cap(static_cast<long long>(h) * wpr, 256), 1, masks), 256, 0, st>>>(mask, h, w, bits,
                                                                                                    any);
  after_launch("k_mask_u8_to_bits");
}

void launch_plan(const uint32_t* bits, int H, int W, int dilate_full, int dilate_scale, int batch,
                 const PlanEntryDev* entries_dev, int num_entries, cudaStream_t st, int per_sample) {
  if (num_entries == 0) return;
  // full-resolution bits + the per-tile-row OR table (tile rows <= 2 H)
  const size_t smem = sizeof(uint32_t) * 3 * H * ((W + 31) >> 5);
  const int use_smem = smem <= 96 * 1024 ? 1 : 0;
  static std::atomic<uint64_t> attr_done{0};
  // (k_plan also has ~140 B of static shared memory: opt in above 47 KB)
  if (use_smem && smem > 47 * 1024 && first_on_device(attr_done))
    SIGE_CUDA(cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
  k_plan<<<num_entries, 1024, use_smem ? smem : 0, st>>>(bits, H, W, dilate_full, dilate_scale,
                                                         batch, entries_dev, use_smem, per_sample);
  after_launch("k_plan");
}

void launch_gn_fold(const Src& x, int groups, float eps, const float* gamma, const float* beta,
                    float* scale, float* shift, double* scratch, int scratch_len, int exact,
                    cudaStream_t st) {
  if (groups < 1 || x.c % groups != 0)
    throw ConfigError("compute_norm_stats: groups " + std::to_string(groups) +
                      " must divide channels " + std::to_string(x.c));
  if (exact) {
    const int items = x.n * groups;
    k_gn_exact<<<(items + 31) / 32, 32, 0, st>>>(x, groups, eps, gamma, beta, scale, shift);
    after_launch("k_gn_exact");
  } else if (scratch && x.c <= 1024 && 2LL * x.n * groups * 2 <= scratch_len) {
    const long long hw = static_cast<long long>(x.h) * x.w;
    int S = static_cast<int>(std::max(1LL, std::min<long long>(hw / 16, (2LL * sm_count()) / x.n)));
    S = static_cast<int>(std::min<long long>(S, scratch_len / (2LL * x.n * groups)));
    const int threads = std::min(1024, std::max(32, (x.c + 31) / 32 * 32));
    k_gn_partial<<<x.n * S, threads, 2 * x.c * sizeof(double), st>>>(x, groups, S, scratch);
    after_launch("k_gn_partial");
    const int items = x.n * x.c;
    k_gn_final<<<(items + 255) / 256, 256, 0, st>>>(x.n * groups, groups, S, x.c,
                                                   static_cast<long long>(x.c / groups) * hw, eps, scratch,
                                                   gamma, beta, scale, shift);
    after_launch("k_gn_final");
  } else {
    k_gn_fast<<<x.n * groups, 512, 0, st>>>(x, groups, eps, gamma, beta, scale, shift);
    after_launch("k_gn_fast");
  }
}

void launch_bn_fold(int c, float eps, const float* gamma, const float* beta, const float* rmean,
                    const float* rvar, float* scale, float* shift, cudaStream_t st) {
  k_bn_fold<<<(c + 255) / 256, 256, 0, st>>>(c, eps, gamma, beta, rmean, rvar, scale, shift);
  after_launch("k_bn_fold");
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  SIGE_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

void launch_materialize_act(const Src& src, void* dst, int half, cudaStream_t st) {
  const long long total = static_cast<long long>(src.n) * src.c * src.h * src.w;
  Src s = src;
  s.epi.fast = 1;  // activation buffers exist in the tensor-core modes only
  k_materialize_act<<<grid_cap(total, 256), 256, 0, st>>>(s, dst, half);
  after_launch("k_materialize_act");
}

void launch_materialize(const Src& src, float* dst, int dst_layout, cudaStream_t st) {
  const long long total = static_cast<long long>(src.n) * src.c * src.h * src.w;
  k_materialize<<<grid_cap(total, 256), 256, 0, st>>>(src, dst, dst_layout);
  after_launch("k_materialize");
}

void launch_tiles_apply(const Src& src, const Tiles& tiles, float* dst, int dst_layout,
                        cudaStream_t st) {
  const long long total = static_cast<long long>(tiles.capacity) * tiles.bh * tiles.bw * src.c;
  if (total == 0) return;
  launch_pdl(k_tiles_apply, dim3(grid_cap(total, 256)), dim3(256), st, src, tiles, dst, dst_layout);
  after_launch("k_tiles_apply");
}

void launch_identity_join(const Src& src, const Tiles& tiles, const Dst& dst, cudaStream_t st) {
  const long long total = static_cast<long long>(tiles.capacity) * tiles.bh * tiles.bw * dst.c;
  if (total == 0) return;
  launch_pdl(k_identity_join, dim3(grid_cap(total, 256)), dim3(256), st, src, tiles, dst);
  after_launch("k_identity_join");
}

void launch_restore(const RestoreJob* jobs_dev, int num_jobs, int max_elems_per_job,
                    cudaStream_t st) {
  if (num_jobs == 0) return;
  // x: tiles of a job (one CTA pass per tile on the channels-last path); y: jobs.
  const int gx = std::max(1, std::min(sm_count() * 4 / std::max(1, num_jobs) + 1, 256));
  (void)max_elems_per_job;
  launch_pdl(k_restore, dim3(gx, num_jobs), dim3(256), st, jobs_dev, 1 << 30);
  after_launch("k_restore");
}

void launch_finalize(const Src& result, const float* cached_final, const int32_t* any, float* out,
                     cudaStream_t st, int per_sample) {
  const long long total = static_cast<long long>(result.n) * result.c * result.h * result.w;
  launch_pdl(k_finalize, dim3(grid_cap(total, 256)), dim3(256), st, result, cached_final, any, out, per_sample);
  after_launch("k_finalize");
}

void launch_add(const float* a, const float* b, float* out, size_t n, cudaStream_t st) {
  launch_add_h(a, b, out, nullptr, n, st);
}

void launch_add_h(const float* a, const float* b, float* out, void* out_h16, size_t n, cudaStream_t st) {
  k_add<<<grid_cap(static_cast<long long>(n), 256), 256, 0, st>>>(a, b, out, static_cast<__half*>(out_h16),
                                                                  static_cast<long long>(n));
  after_launch("k_add");
}

void launch_input_twin(const float* in, int n, int c, int h, int w, int c_pad, void* out, cudaStream_t st) {
  const long long total = static_cast<long long>(n) * h * w * c_pad;
  launch_pdl(k_input_twin, dim3(grid_cap(total, 256)), dim3(256), st, in, n, c, h, w, c_pad,
             static_cast<__half*>(out));
  after_launch("k_input_twin");
}

void launch_to_half(const float* src, void* dst_h16, size_t n, cudaStream_t st) {
  k_to_half<<<grid_cap(static_cast<long long>(n), 256), 256, 0, st>>>(src, static_cast<__half*>(dst_h16),
                                                                      static_cast<long long>(n));
  after_launch("k_to_half");
}

void launch_nchw_to_nhwc(const float* in, float* out, int n, int c, int h, int w, cudaStream_t st) {
  k_nchw_to_nhwc<<<grid_cap(static_cast<long long>(n) * c * h * w, 256), 256, 0, st>>>(in, out, n, c, h, w);
  after_launch("k_nchw_to_nhwc");
}

void launch_nhwc_to_nchw(const float* in, float* out, int n, int c, int h, int w, cudaStream_t st) {
  k_nhwc_to_nchw<<<grid_cap(static_cast<long long>(n) * c * h * w, 256), 256, 0, st>>>(in, out, n, c, h, w);
  after_launch("k_nhwc_to_nchw");
}

void launch_resize_nhwc(const float* in, int n, int c, int H, int W, int h, int w, float* out, void* out16, int c16,
                        cudaStream_t st) {
  const long long total = static_cast<long long>(n) * h * w * c16;
  launch_pdl(k_resize_nhwc, dim3(grid_cap(total, 256)), dim3(256), st, in, n, c, H, W, h, w, out,
             static_cast<__half*>(out16), c16);
  after_launch("k_resize_nhwc");
}

void launch_spade_mod(const Src& x, const float* sc, const float* sh, const float* gb, int act, const Tiles* tiles,
                      float* out, void* out16, cudaStream_t st) {
  Tiles t{};
  long long total = static_cast<long long>(x.n) * x.h * x.w * x.c;
  if (tiles) {
    t = *tiles;
    total = static_cast<long long>(t.capacity) * t.bh * t.bw * x.c;
  }
  if (total == 0) return;
  launch_pdl(k_spade_mod, dim3(grid_cap(total, 256)), dim3(256), st, x, sc, sh, gb, act, t, out,
             static_cast<__half*>(out16));
  after_launch("k_spade_mod");
}

}  // namespace sige_b200
