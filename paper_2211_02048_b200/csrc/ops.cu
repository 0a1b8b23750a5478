// ops.cu — op-level sm_100a kernels: the per-function drop-ins for
// proj/include/sige/{mask,kernels,conv}.hpp. Layouts are the reference's
// (NCHW tensors, (G,C,bh,bw) block stacks, {n,r,c} index triplets). These are
// HBM-bound copies / predicates; float arithmetic uses __f*_rn intrinsics so
// no FMA contraction happens and results are bit-exact to the reference.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "common.hpp"
#include "ops.hpp"

#include <cstdlib>

namespace sige_b200 {

namespace {

constexpr int kThreads = 256;

inline int grid_for(long long n, int threads = kThreads) {
  long long g = (n + threads - 1) / threads;
  long long cap = static_cast<long long>(sm_count()) * 32;
  return static_cast<int>(g < 1 ? 1 : (g > cap ? cap : g));
}

// ---------------------------------------------------------------- masks --

// compute_difference_mask (mask.cpp:14-32): mask[p] |= |e - o| > t over all
// (n, c) planes. Grid.y splits the planes; writers only ever store 1, so
// concurrent stores to one byte are benign.
__global__ void k_difference_mask(const float* __restrict__ o, const float* __restrict__ e,
                                  int planes, int planes_per_y, long long hw, float thr,
                                  uint8_t* __restrict__ mask) {
  int p0 = blockIdx.y * planes_per_y;
  int p1 = min(planes, p0 + planes_per_y);
  const bool vec = (hw & 3) == 0 && ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(e)) & 15) == 0;
  long long nq = vec ? hw / 4 : hw;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nq;
       q += (long long)gridDim.x * blockDim.x) {
    if (vec) {
      bool b0 = false, b1 = false, b2 = false, b3 = false;
      for (int p = p0; p < p1; ++p) {
        float4 a = __ldg(reinterpret_cast<const float4*>(o + p * hw) + q);
        float4 b = __ldg(reinterpret_cast<const float4*>(e + p * hw) + q);
        b0 |= fabsf(__fsub_rn(b.x, a.x)) > thr;
        b1 |= fabsf(__fsub_rn(b.y, a.y)) > thr;
        b2 |= fabsf(__fsub_rn(b.z, a.z)) > thr;
        b3 |= fabsf(__fsub_rn(b.w, a.w)) > thr;
      }
      if (b0) mask[4 * q] = 1;
      if (b1) mask[4 * q + 1] = 1;
      if (b2) mask[4 * q + 2] = 1;
      if (b3) mask[4 * q + 3] = 1;
    } else {
      bool any = false;
      for (int p = p0; p < p1; ++p)
        any |= fabsf(__fsub_rn(__ldg(e + p * hw + q), __ldg(o + p * hw + q))) > thr;
      if (any) mask[q] = 1;
    }
  }
}

// downsample_mask (mask.cpp:34-53): max-pool by integer factors.
__global__ void k_downsample_mask(const uint8_t* __restrict__ m, int h, int w, int oh, int ow,
                                  uint8_t* __restrict__ out) {
  int fy = h / oh, fx = w / ow;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < oh * ow; p += gridDim.x * blockDim.x) {
    int y = p / ow, x = p % ow;
    uint8_t v = 0;
    for (int dy = 0; dy < fy && !v; ++dy)
      for (int dx = 0; dx < fx && !v; ++dx) v = m[(size_t)(y * fy + dy) * w + x * fx + dx];
    out[p] = v ? 1 : 0;
  }
}

// dilate_mask (mask.cpp:55-80): separable Chebyshev dilation, clipped.
__global__ void k_dilate_rows(const uint8_t* __restrict__ m, int h, int w, int r,
                              uint8_t* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < h * w; p += gridDim.x * blockDim.x) {
    int y = p / w, x = p % w;
    uint8_t v = 0;
    for (int t = max(0, x - r); t <= min(w - 1, x + r) && !v; ++t) v = m[(size_t)y * w + t];
    out[p] = v ? 1 : 0;
  }
}
__global__ void k_dilate_cols(const uint8_t* __restrict__ m, int h, int w, int r,
                              uint8_t* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < h * w; p += gridDim.x * blockDim.x) {
    int y = p / w, x = p % w;
    uint8_t v = 0;
    for (int t = max(0, y - r); t <= min(h - 1, y + r) && !v; ++t) v = m[(size_t)t * w + x];
    out[p] = v ? 1 : 0;
  }
}

// mask_to_block_indices (mask.cpp:103-136). One CTA walks the tile grid in
// row-major chunks of blockDim tiles; each thread tests one tile, a block
// scan assigns output slots, so the emitted order is exactly the reference's
// (r outer, c inner), then replicated n-major.
__global__ void k_blockify(const uint8_t* __restrict__ m, int h, int w, int b, int batch,
                           int32_t* __restrict__ idx, int capacity, int32_t* __restrict__ count) {
  __shared__ int warp_sums[32];
  __shared__ int base;
  int ty = (h + b - 1) / b, tx = (w + b - 1) / b, tiles = ty * tx;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int t0 = 0; t0 < tiles; t0 += blockDim.x) {
    int t = t0 + threadIdx.x;
    bool on = false;
    int R = 0, Cc = 0;
    if (t < tiles) {
      R = (t / tx) * b;
      Cc = (t % tx) * b;
      for (int y = R; y < min(h, R + b) && !on; ++y)
        for (int x = Cc; x < min(w, Cc + b) && !on; ++x) on = m[(size_t)y * w + x] != 0;
    }
    unsigned bal = __ballot_sync(0xffffffffu, on);
    if (lane == 0) warp_sums[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? warp_sums[lane] : 0;
      for (int d = 1; d < 32; d <<= 1) {
        int u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += u;
      }
      if (lane < nw) warp_sums[lane] = v;  // inclusive
    }
    __syncthreads();
    int before = (wid ? warp_sums[wid - 1] : 0) + __popc(bal & ((1u << lane) - 1u));
    int slot = base + before;
    int total_chunk = warp_sums[nw - 1];
    // Sample 0 first (the tile total is unknown until the walk ends); the
    // other samples are replicated from it below.
    if (on && slot < capacity) {
      idx[3 * slot] = 0;
      idx[3 * slot + 1] = R;
      idx[3 * slot + 2] = Cc;
    }
    __syncthreads();
    if (threadIdx.x == 0) base += total_chunk;
    __syncthreads();
  }
  int per = base;
  // replicate n-major: entries [per * n, per * (n + 1)) copy sample 0 with n.
  for (int n = 1; n < batch; ++n)
    for (int i = threadIdx.x; i < per; i += blockDim.x) {
      int d = n * per + i;
      if (d < capacity && i < capacity) {
        idx[3 * d] = n;
        idx[3 * d + 1] = idx[3 * i + 1];
        idx[3 * d + 2] = idx[3 * i + 2];
      }
    }
  if (threadIdx.x == 0) *count = per * batch;
}

// ---------------------------------------------------------------- blocks --

// scatter (kernels.cpp:88-132) moves a CHUNK of consecutive tiles x a slice
// of channels per CTA pass through shared memory, so both sides are
// coalesced: the block-stack side as one contiguous run per tile, the image
// side walked in (channel, row, tile, column) order — the index set is
// row-major (mask.cpp:103-136), so a chunk's tiles are mostly horizontal
// neighbours and a warp's b-wide tile rows merge into full-line stores.
// Non-adjacent tiles stay correct, only less coalesced. Tiles larger than the
// staging buffer fall back to a direct walk (staged = false). (The same
// staging for gather measured slower than gather's per-tile walk below:
// 114-250 us vs 100 us at the ops_hbm workload, profiles/r1_ops_hbm_iter.txt.)
constexpr int kChunkCols = 256;  // image-side columns (tiles x tile width) per chunk
constexpr int kMaxChunkTiles = 256;
constexpr int kStageFloats = 8192;  // 32 KB staging buffer per CTA
constexpr int kU = 8;               // independent loads in flight per thread

struct ChunkPlan {
  int T;    // tiles per chunk
  int cpi;  // channels per item
  bool staged;
};

inline ChunkPlan chunk_plan(int c, int width) {
  const int wsz = width * width;
  ChunkPlan cp{};
  cp.staged = wsz <= kStageFloats;
  cp.T = std::max(1, std::min(kMaxChunkTiles, kChunkCols / width));
  if (cp.staged) cp.T = std::max(1, std::min(cp.T, kStageFloats / wsz));
  const int cap = cp.staged ? kStageFloats : 4096;
  cp.cpi = std::max(1, std::min(c, cap / (cp.T * wsz)));
  return cp;
}

__device__ __forceinline__ void load_origins(int (*s_org)[3], const int32_t* __restrict__ idx, int i0, int tc,
                                             int stride, int pad) {
  __syncthreads();
  for (int t = threadIdx.x; t < tc; t += blockDim.x) {
    s_org[t][0] = __ldg(idx + 3 * (i0 + t));
    s_org[t][1] = __ldg(idx + 3 * (i0 + t) + 1) * stride - pad;
    s_org[t][2] = __ldg(idx + 3 * (i0 + t) + 2) * stride - pad;
  }
  __syncthreads();
}

// Column walk of the scatter: the image side of an item is a grid of
// rows (channel, tile row) x cols (tile, tile column). A thread owns one
// column (one division per column and item) and a strided set of channels,
// and walks each channel's tile rows with plain pointer arithmetic — no
// per-element division (integer issue, not bandwidth, bounded a version that
// decoded every element's coordinates).
struct ColWalk {
  int groups, group, col, col_step;
  __device__ ColWalk(int cols) {
    groups = cols >= static_cast<int>(blockDim.x) ? 1 : static_cast<int>(blockDim.x) / cols;
    group = groups > 1 ? static_cast<int>(threadIdx.x) / cols : 0;
    col = groups > 1 ? static_cast<int>(threadIdx.x) - group * cols : static_cast<int>(threadIdx.x);
    col_step = groups > 1 ? cols : static_cast<int>(blockDim.x);
    if (group >= groups) col = cols;  // spare threads
  }
};

// Contiguous per-tile runs of a block stack (tile t's `run` floats at
// stack + t * slab) into shared memory (sbuf + t * run), 16-byte vectors when
// the geometry keeps them aligned.
__device__ __forceinline__ void stack_to_smem_issue(const float* stack, size_t slab, float* sbuf, int tc, int run,
                                                    bool vec) {
  const int v = vec ? 4 : 1, rv = run / v;
  const int tpp = rv >= static_cast<int>(blockDim.x) ? 1 : static_cast<int>(blockDim.x) / rv;
  int t = tpp > 1 ? static_cast<int>(threadIdx.x) / rv : 0;
  const int j0 = tpp > 1 ? static_cast<int>(threadIdx.x) - t * rv : static_cast<int>(threadIdx.x);
  const int jstep = tpp > 1 ? rv : static_cast<int>(blockDim.x);
  if (t >= tpp) return;
  for (; t < tc; t += tpp) {
    const float* g = stack + t * slab;
    float* sm = sbuf + t * run;
    for (int j = j0; j < rv; j += jstep) {
      // cp.async: no register round trip per copy, so all of a thread's
      // copies are in flight at once (a dependent ld -> st per iteration
      // left ~1 load per thread outstanding: latency-bound staging)
      const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(vec ? sm + 4 * j : sm + j));
      if (vec)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(g + 4 * j) : "memory");
      else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(g + j) : "memory");
    }
  }
}
__device__ __forceinline__ void stack_to_smem(const float* stack, size_t slab, float* sbuf, int tc, int run,
                                              bool vec) {
  stack_to_smem_issue(stack, slab, sbuf, tc, run, vec);
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// gather (kernels.cpp:39-86): one thread per output value; out-of-canvas
// cells are +0 and skip the epilogue.
__global__ void k_gather(const float* __restrict__ x, int c, int h, int w,
                         const int32_t* __restrict__ idx, int count, int win, int stride, int pad,
                         DevEpilogue epi, float* __restrict__ out) {
  // One tile per blockIdx.x (grid-stride). A thread owns quads (4 consecutive
  // outputs of the tile slab (C, win, win), indices advanced incrementally,
  // one 16-byte store each) and keeps two quads = 8 loads in flight.
  constexpr int kQ = 2;
  const int wsz = win * win, slab = c * wsz;
  const bool vec = (slab & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (int i = blockIdx.x; i < count; i += gridDim.x) {
    const int n = __ldg(idx + 3 * i), oy = __ldg(idx + 3 * i + 1) * stride - pad,
              ox = __ldg(idx + 3 * i + 2) * stride - pad;
    const size_t plane0 = static_cast<size_t>(n) * c;
    float* o = out + static_cast<size_t>(i) * slab;
    for (int q0 = threadIdx.x * 4; q0 < slab; q0 += blockDim.x * 4 * kQ) {
      float v[kQ][4];
#pragma unroll
      for (int k = 0; k < kQ; ++k) {
        const int q = q0 + k * blockDim.x * 4;
        int ch = q / wsz, cell = q - ch * wsz;
        int wy = cell / win, wx = cell - wy * win;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          v[k][e] = 0.0f;
          if (q + e < slab) {
            const int sy = oy + wy, sx = ox + wx;
            if (sy >= 0 && sy < h && sx >= 0 && sx < w) {
              v[k][e] = __ldg(x + ((plane0 + ch) * h + sy) * w + sx);
              if (epi.num_steps) v[k][e] = dev_epi(epi, v[k][e], ch, c, n);
            }
          }
          if (++wx == win) {
            wx = 0;
            if (++wy == win) {
              wy = 0;
              ++ch;
            }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kQ; ++k) {
        const int q = q0 + k * blockDim.x * 4;
        if (q >= slab) break;
        if (vec)
          *reinterpret_cast<float4*>(o + q) = make_float4(v[k][0], v[k][1], v[k][2], v[k][3]);
        else
          for (int e = 0; e < 4 && q + e < slab; ++e) o[q + e] = v[k][e];
      }
    }
  }
}

// gather, row form (W % 4 == 0, win in {4, 8}): one thread per window row
// (tile, channel, row) — the row's source span is read as the 16-byte aligned
// float4 chunks that cover it (chunks never straddle an image row when
// W % 4 == 0; chunks outside the canvas stay zero) and written as win/4
// 16-byte stores. Same values as k_gather (zero fill, the chain on in-canvas
// cells only); ~4x fewer memory instructions per element. (A tile-fastest
// order — coalesced reads across adjacent tiles, scattered 32-byte writes —
// measured 94 vs 90 us at the ops_hbm workload.)
template <int WIN>
__global__ void __launch_bounds__(256) k_gather_rows(const float* __restrict__ x, int c, int h, int w,
                                                     const int32_t* __restrict__ idx, int count, long long rows,
                                                     int stride, int pad, DevEpilogue epi, float* __restrict__ out) {
  constexpr int kChunks = WIN / 4 + 1;  // aligned float4 chunks covering WIN floats at any phase
  // warp-uniform trip count (the tile origin is fetched once per warp when
  // the warp's rows share a tile: the LSU data pipe, not DRAM, bounds this kernel)
  const int lane = threadIdx.x & 31;
  for (long long rb = blockIdx.x * static_cast<long long>(blockDim.x) + (threadIdx.x & ~31); rb < rows;
       rb += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = rb + lane;
    if (r >= rows) continue;  // (tail warp: no shuffles below depend on inactive lanes)
    const int wy = static_cast<int>(r % WIN);
    const long long gc = r / WIN;  // tile * c + channel (the output is written in order)
    const int ch = static_cast<int>(gc % c);
    const int i = static_cast<int>(gc / c);
    const unsigned act = __activemask();
    const int i0 = __shfl_sync(act, i, __ffs(act) - 1);
    int n, oy, ox;
    if ((act & 7u) == 7u && __all_sync(act, i == i0)) {  // lanes 0-2 fetch (n, y, x)
      const int v = lane < 3 ? __ldg(idx + 3 * i0 + lane) : 0;
      n = __shfl_sync(act, v, 0), oy = __shfl_sync(act, v, 1), ox = __shfl_sync(act, v, 2);
    } else {
      n = __ldg(idx + 3 * i), oy = __ldg(idx + 3 * i + 1), ox = __ldg(idx + 3 * i + 2);
    }
    const int sy = oy * stride - pad + wy, sx0 = ox * stride - pad;
    float v[WIN];
#pragma unroll
    for (int k = 0; k < WIN; ++k) v[k] = 0.0f;
    if (sy >= 0 && sy < h) {
      const float* row = x + ((static_cast<size_t>(n) * c + ch) * h + sy) * w;
      const int base = sx0 & ~3;  // aligned start (sx0 may be negative)
      const int ph = sx0 - base;  // 0..3
      float buf[kChunks * 4];
#pragma unroll
      for (int q = 0; q < kChunks; ++q) {
        const int xs = base + 4 * q;
        float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
        if (xs >= 0 && xs < w) f = __ldg(reinterpret_cast<const float4*>(row + xs));
        buf[4 * q] = f.x, buf[4 * q + 1] = f.y, buf[4 * q + 2] = f.z, buf[4 * q + 3] = f.w;
      }
      // v[k] = buf[ph + k] with compile-time indices only (a runtime-indexed
      // register array would live in local memory)
#pragma unroll
      for (int k = 0; k < WIN; ++k)
        v[k] = ph == 0 ? buf[k] : ph == 1 ? buf[k + 1] : ph == 2 ? buf[k + 2] : buf[k + 3];
      if (epi.num_steps) {
#pragma unroll
        for (int k = 0; k < WIN; ++k) {
          const int sx = sx0 + k;
          if (sx >= 0 && sx < w) v[k] = dev_epi(epi, v[k], ch, c, n);
        }
      }
    }
    float4* o = reinterpret_cast<float4*>(out + ((static_cast<size_t>(i) * c + ch) * WIN + wy) * WIN);
#pragma unroll
    for (int k = 0; k < WIN; k += 4) o[k / 4] = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
  }
}

// gather, 8-wide window rows with 256-bit loads (sm_100 LDG.256): the row
// form above is bound by L1 LSU wavefronts (one per touched line per load
// instruction); two 32-byte-aligned loads cover 8 floats at any phase where
// the row form needs three 16-byte ones. Needs w % 8 == 0 and a 32-byte
// aligned x (checked on the host).
__device__ __forceinline__ void ldg256(const float* p, float* v) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__global__ void __launch_bounds__(256) k_gather_rows8w(const float* __restrict__ x, int c, int h, int w,
                                                       const int32_t* __restrict__ idx, int count, long long rows,
                                                       int stride,
                                                       int pad, DevEpilogue epi, float* __restrict__ out) {
  constexpr int WIN = 8;
  const int lane = threadIdx.x & 31;
  const bool st256 = (reinterpret_cast<uintptr_t>(out) & 31) == 0;  // one 256-bit store per row
  for (long long rb = blockIdx.x * static_cast<long long>(blockDim.x) + (threadIdx.x & ~31); rb < rows;
       rb += static_cast<long long>(gridDim.x) * blockDim.x) {
    // a warp = 4 consecutive tiles (usually horizontal neighbours) x 8 window
    // rows of one channel: each load instruction touches ~16 lines instead of
    // the 32 of a one-tile warp (the LSU data pipe bounds this kernel)
    const long long r = rb + lane;
    if (r >= rows) continue;
    const int wy = static_cast<int>(r & 7), j = static_cast<int>((r >> 3) & 3);
    const long long gq = r >> 5;  // tile quad * c + channel
    const int ch = static_cast<int>(gq % c);
    const int i = static_cast<int>(gq / c) * 4 + j;
    const unsigned act = __activemask();
    const int t0 = (static_cast<int>(gq / c)) * 4;
    int n, oy, ox;
    if (act == 0xffffffffu && t0 + 4 <= count) {  // lanes 0-11 fetch the quad's origins
      const int v = lane < 12 ? __ldg(idx + 3 * t0 + lane) : 0;
      n = __shfl_sync(act, v, 3 * j), oy = __shfl_sync(act, v, 3 * j + 1), ox = __shfl_sync(act, v, 3 * j + 2);
    } else {
      if (i >= count) continue;
      n = __ldg(idx + 3 * i), oy = __ldg(idx + 3 * i + 1), ox = __ldg(idx + 3 * i + 2);
    }
    const int sy = oy * stride - pad + wy, sx0 = ox * stride - pad;
    float v[WIN];
#pragma unroll
    for (int k = 0; k < WIN; ++k) v[k] = 0.0f;
    if (sy >= 0 && sy < h) {
      const float* row = x + ((static_cast<size_t>(n) * c + ch) * h + sy) * w;
      const int base = sx0 & ~7;  // 32-byte aligned start (sx0 may be negative)
      const int ph = sx0 - base;  // 0..7
      float buf[16];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int xs = base + 8 * q;
        if (xs >= 0 && xs < w && (q == 0 || ph > 0)) {
          ldg256(row + xs, buf + 8 * q);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) buf[8 * q + k] = 0.0f;
        }
      }
      // v[k] = buf[ph + k]: a 3-stage barrel shift (compile-time indices only)
      if (ph & 4) {
#pragma unroll
        for (int k = 0; k < 12; ++k) buf[k] = buf[k + 4];
      }
      if (ph & 2) {
#pragma unroll
        for (int k = 0; k < 10; ++k) buf[k] = buf[k + 2];
      }
      if (ph & 1) {
#pragma unroll
        for (int k = 0; k < 9; ++k) buf[k] = buf[k + 1];
      }
#pragma unroll
      for (int k = 0; k < WIN; ++k) v[k] = buf[k];
      if (epi.num_steps) {
#pragma unroll
        for (int k = 0; k < WIN; ++k) {
          const int sx = sx0 + k;
          if (sx >= 0 && sx < w) v[k] = dev_epi(epi, v[k], ch, c, n);
        }
      }
    }
    float* o = out + ((static_cast<size_t>(i) * c + ch) * WIN + wy) * WIN;
    if (st256) {
      asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(o), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                   "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                   : "memory");
    } else {
      reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(o)[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
}

// scatter_inplace / scatter_add_inplace: tile values clipped at the fringe;
// mode 0 writes, mode 1 adds.
__global__ void __launch_bounds__(kThreads) k_scatter(const float* __restrict__ blocks, int count, int c, int b,
                                                      const int32_t* __restrict__ idx, float* __restrict__ base,
                                                      int nsamp, int h, int w, int T, int cpi, int staged, int mode,
                                                      int pairs) {
  __shared__ int s_org[kMaxChunkTiles][3];
  __shared__ __align__(16) float s_buf[kStageFloats];
  const int bsz = b * b;
  const size_t slab = static_cast<size_t>(c) * bsz, plane = static_cast<size_t>(h) * w;
  const int chunks = (count + T - 1) / T, slices = (c + cpi - 1) / cpi;
  for (int it = blockIdx.x; it < chunks * slices; it += gridDim.x) {
    const int ck = it / slices, c0 = (it - ck * slices) * cpi, ncl = min(c, c0 + cpi) - c0;
    const int i0 = ck * T, tc = min(T, count - i0);
    load_origins(s_org, idx, i0, tc, 1, 0);
    const float* sb = blocks + static_cast<size_t>(i0) * slab + static_cast<size_t>(c0) * bsz;
    const int run = ncl * bsz;
    if (staged) {
      stack_to_smem(sb, slab, s_buf, tc, run, (bsz & 3) == 0 && (reinterpret_cast<uintptr_t>(blocks) & 15) == 0);
      __syncthreads();
    }
    // image side: rows (channel, tile row), cols (tile, tile column). With
    // an even block and width a thread owns a column PAIR (8-byte stores, the
    // pairs never straddle the image edge): half the store instructions.
    if (pairs) {
      // (a whole 6-wide tile row per thread measured slower: 88 vs 68 us)
      const int per = 2, hb = b / per, pcols = tc * hb;
      ColWalk pw(pcols);
      for (; pw.col < pcols; pw.col += pw.col_step) {
        const int t = pw.col / hb, dx = (pw.col - t * hb) * per;
        const int y0 = s_org[t][1], xx = s_org[t][2] + dx;
        const bool inside = s_org[t][0] >= 0 && s_org[t][0] < nsamp && y0 >= 0 && s_org[t][2] >= 0;
        const int dy_hi = inside && xx < w ? min(b, h - y0) : 0;
        float* dpb = base + (static_cast<size_t>(s_org[t][0]) * c + c0) * plane + static_cast<size_t>(y0) * w + xx;
        const float* sp = s_buf + t * run + dx;
        for (int cl = pw.group; cl < ncl; cl += pw.groups) {
          float* dc = dpb + static_cast<size_t>(cl) * plane;
          const float* sc = sp + cl * bsz;
#pragma unroll 6
          for (int dy = 0; dy < dy_hi; ++dy) {
            for (int q = 0; q < per; q += 2) {  // (a 6-wide row: the width check keeps the fringe)
              if (xx + q >= w) break;
              float2 v = *reinterpret_cast<const float2*>(sc + dy * b + q);
              if (mode) {
                const float2 cur = *reinterpret_cast<const float2*>(dc + dy * w + q);
                v.x = __fadd_rn(cur.x, v.x);
                v.y = __fadd_rn(cur.y, v.y);
              }
              *reinterpret_cast<float2*>(dc + dy * w + q) = v;
            }
          }
        }
      }
      continue;
    }
    const int cols = tc * b;
    ColWalk cw(cols);
    for (; cw.col < cols; cw.col += cw.col_step) {
      const int t = cw.col / b, dx = cw.col - t * b;
      const int y0 = s_org[t][1], xx = s_org[t][2] + dx;
      // fringe clipping; an index outside the tensor (the wrappers reject it,
      // require_scatter_compatible, kernels.cpp:18-35) never writes
      const bool inside = s_org[t][0] >= 0 && s_org[t][0] < nsamp && y0 >= 0 && s_org[t][2] >= 0;
      const int dy_hi = inside && xx < w ? min(b, h - y0) : 0;
      float* dpb = base + (static_cast<size_t>(s_org[t][0]) * c + c0) * plane + static_cast<size_t>(y0) * w + xx;
      const float* sp = staged ? s_buf + t * run + dx : sb + t * slab + dx;
      for (int cl = cw.group; cl < ncl; cl += cw.groups) {
        float* dc = dpb + static_cast<size_t>(cl) * plane;
        const float* sc = sp + cl * bsz;
        if (mode) {
#pragma unroll 4
          for (int dy = 0; dy < dy_hi; ++dy) dc[dy * w] = __fadd_rn(dc[dy * w], staged ? sc[dy * b] : __ldg(sc + dy * b));
        } else {
#pragma unroll 8
          for (int dy = 0; dy < dy_hi; ++dy) dc[dy * w] = staged ? sc[dy * b] : __ldg(sc + dy * b);
        }
      }
    }
  }
}

// scatter with the staging double-buffered (a persistent CTA stages item
// i + 1 with cp.async while it stores item i): the staged column-pair walk of
// k_scatter (above) behind a two-deep copy pipeline. Item = (chunk of T tiles,
// slice of cpi channels); the stack side of an item is T runs of cpi * b^2
// contiguous floats, the origins 3 T contiguous ints.
constexpr int kPipeFloats = 6144;     // per buffer (two buffers in dynamic shared memory: 48 KB)
constexpr int kPipeMaxFloats = 16384;  // SIGE_SCATTER_STAGE cap
__global__ void __launch_bounds__(kThreads) k_scatter_pipe(const float* __restrict__ blocks, int count, int c,
                                                           int b, const int32_t* __restrict__ idx,
                                                           float* __restrict__ base, int nsamp, int h, int w,
                                                           int T, int cpi, int mode, int buf_floats) {
  __shared__ __align__(16) int s_org[2][kMaxChunkTiles * 3];
  extern __shared__ __align__(16) float s_dyn[];
  const int bsz = b * b;
  const size_t slab = static_cast<size_t>(c) * bsz, plane = static_cast<size_t>(h) * w;
  const int chunks = (count + T - 1) / T, slices = (c + cpi - 1) / cpi, items = chunks * slices;
  const bool vec = (bsz & 3) == 0 && (reinterpret_cast<uintptr_t>(blocks) & 15) == 0;
  // items advance by gridDim.x: (chunk, slice) stepped without divisions
  const int dq = gridDim.x / slices, dr = gridDim.x - dq * slices;
  auto step = [&](int& ck, int& sl) {
    ck += dq, sl += dr;
    if (sl >= slices) sl -= slices, ++ck;
  };
  // the column walk of a full chunk, decoded once (this kernel is issue-bound)
  const int per = (b & 1) == 0 && (w & 1) == 0 && (reinterpret_cast<uintptr_t>(base) & 7) == 0 ? 2 : 1, hb = b / per;
  const ColWalk pw_full(T * hb);
  const int t_full = pw_full.col / hb;
  auto issue = [&](int ck, int sl, int sbi) {
    const int c0 = sl * cpi, ncl = min(c, c0 + cpi) - c0;
    const int i0 = ck * T, tc = min(T, count - i0);
    for (int j = threadIdx.x; j < 3 * tc; j += blockDim.x) {
      const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(&s_org[sbi][j]));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(idx + 3 * i0 + j) : "memory");
    }
    stack_to_smem_issue(blocks + static_cast<size_t>(i0) * slab + static_cast<size_t>(c0) * bsz, slab,
                        s_dyn + sbi * buf_floats, tc, ncl * bsz, vec);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int sbi = 0;
  int ck = blockIdx.x / slices, sl = blockIdx.x - (blockIdx.x / slices) * slices;
  if (blockIdx.x < items) issue(ck, sl, 0);
  for (int it = blockIdx.x; it < items; it += gridDim.x, sbi ^= 1, step(ck, sl)) {
    if (it + static_cast<int>(gridDim.x) < items) {
      int nck = ck, nsl = sl;
      step(nck, nsl);
      issue(nck, nsl, sbi ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const int c0 = sl * cpi, ncl = min(c, c0 + cpi) - c0;
    const int i0 = ck * T, tc = min(T, count - i0), run = ncl * bsz;
    const int* org = s_org[sbi];
    const float* buf = s_dyn + sbi * buf_floats;
    // column pairs (8-byte stores) when the block and width are even
    const int pcols = tc * hb;
    ColWalk pw = tc == T ? pw_full : ColWalk(pcols);
    int t = tc == T ? t_full : pw.col / hb;
    for (; pw.col < pcols;) {
      const int dx = (pw.col - t * hb) * per;
      const int y0 = org[3 * t + 1], xx = org[3 * t + 2] + dx;
      // fringe clipping; an index outside the tensor never writes
      const bool inside = org[3 * t] >= 0 && org[3 * t] < nsamp && y0 >= 0 && org[3 * t + 2] >= 0;
      const int dy_hi = inside && xx < w ? min(b, h - y0) : 0;
      float* dpb = base + (static_cast<size_t>(org[3 * t]) * c + c0) * plane + static_cast<size_t>(y0) * w + xx;
      const float* sp = buf + t * run + dx;
      for (int cl = pw.group; cl < ncl; cl += pw.groups) {
        float* dc = dpb + static_cast<size_t>(cl) * plane;
        const float* sc = sp + cl * bsz;
        if (per == 2) {
#pragma unroll 6
          for (int dy = 0; dy < dy_hi; ++dy) {
            float2 v = *reinterpret_cast<const float2*>(sc + dy * b);
            if (mode) {
              const float2 cur = *reinterpret_cast<const float2*>(dc + dy * w);
              v.x = __fadd_rn(cur.x, v.x);
              v.y = __fadd_rn(cur.y, v.y);
            }
            *reinterpret_cast<float2*>(dc + dy * w) = v;
          }
        } else {
#pragma unroll 4
          for (int dy = 0; dy < dy_hi; ++dy) dc[dy * w] = mode ? __fadd_rn(dc[dy * w], sc[dy * b]) : sc[dy * b];
        }
      }
      pw.col += pw.col_step;
      if (pw.col < pcols) t = pw.col / hb;
    }
    __syncthreads();  // buffer sbi is refilled by the next iteration's issue
  }
}

// SPADE modulation gather (config 3; restated in orc_gather_spade): gather's
// per-tile walk (above) with v -> norm chain -> v * (1 + gamma) + beta -> act
// on in-canvas cells, each operation rounded separately (bit-exact to the
// restatement).
__device__ __forceinline__ float spade_act(float v, int act, int fma_expf) {
  if (act == SIGE_ACT_LEAKY_RELU) return v > 0.0f ? v : __fmul_rn(0.2f, v);
  return dev_act(v, act, fma_expf);
}

__global__ void k_gather_spade(const float* __restrict__ x, const float* __restrict__ gamma,
                               const float* __restrict__ beta, int c, int h, int w,
                               const int32_t* __restrict__ idx, int count, int win, int stride, int pad,
                               DevEpilogue epi, int act, float* __restrict__ out) {
  const int wsz = win * win, slab = c * wsz;
  for (int i = blockIdx.x; i < count; i += gridDim.x) {
    const int n = __ldg(idx + 3 * i), oy = __ldg(idx + 3 * i + 1) * stride - pad,
              ox = __ldg(idx + 3 * i + 2) * stride - pad;
    float* o = out + static_cast<size_t>(i) * slab;
    for (int q = threadIdx.x; q < slab; q += blockDim.x) {
      const int ch = q / wsz, cell = q - ch * wsz, wy = cell / win, wx = cell - wy * win;
      const int sy = oy + wy, sx = ox + wx;
      float v = 0.0f;
      if (sy >= 0 && sy < h && sx >= 0 && sx < w) {
        const size_t at = ((static_cast<size_t>(n) * c + ch) * h + sy) * w + sx;
        v = __ldg(x + at);
        if (epi.num_steps) v = dev_epi(epi, v, ch, c, n);
        v = __fmul_rn(v, __fadd_rn(1.0f, __ldg(gamma + at)));
        v = __fadd_rn(v, __ldg(beta + at));
        v = spade_act(v, act, epi.fma_expf);
      }
      o[q] = v;
    }
  }
}

__global__ void k_resize_nearest(const float* __restrict__ in, long long planes, int h, int w, int oh, int ow,
                                 float* __restrict__ out) {
  const long long total = planes * oh * ow;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = static_cast<int>(e % ow);
    const long long r = e / ow;
    const int y = static_cast<int>(r % oh);
    const long long p = r / oh;
    const int sy = oh <= h ? y * (h / oh) : y / (oh / h), sx = ow <= w ? x * (w / ow) : x / (ow / w);
    out[e] = __ldg(in + (p * h + sy) * w + sx);
  }
}

__global__ void k_map_fill(sige_scatter_entry* map, long long hw) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < hw;
       p += (long long)gridDim.x * blockDim.x) {
    sige_scatter_entry e;
    e.block = -1;
    e.dy = 0;
    e.dx = 0;
    map[p] = e;
  }
}
__global__ void k_map_tiles(const int32_t* __restrict__ idx, int per, int b, int h, int w,
                            sige_scatter_entry* map) {
  long long total = (long long)per * b * b;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    int o = static_cast<int>(q / (b * b));
    int cell = static_cast<int>(q % (b * b));
    int dy = cell / b, dx = cell % b;
    int y = idx[3 * o + 1] + dy, x = idx[3 * o + 2] + dx;
    if (y >= h || x >= w) continue;
    sige_scatter_entry e;
    e.block = o;
    e.dy = static_cast<int16_t>(dy);
    e.dx = static_cast<int16_t>(dx);
    map[(size_t)y * w + x] = e;
  }
}
// per-sample count and batch-pattern check (kernels.cpp:142-152).
__global__ void k_map_check(const int32_t* __restrict__ idx, int count, int* out) {
  // out[0] = per-sample count, out[1] = 1 if the pattern differs.
  __shared__ int per_s;
  if (threadIdx.x == 0) per_s = 0;
  __syncthreads();
  int local = 0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) local += idx[3 * i] == idx[0];
  atomicAdd(&per_s, local);
  __syncthreads();
  int per = per_s;
  int bad = 0;
  if (per > 0)
    for (int i = per + threadIdx.x; i < count; i += blockDim.x) {
      int r = i % per;
      bad |= idx[3 * i + 1] != idx[3 * r + 1] || idx[3 * i + 2] != idx[3 * r + 2];
    }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    out[0] = per;
    out[1] = bad;
  }
}

// scatter_gather (kernels.cpp:204-275).
__global__ void k_scatter_gather(const float* __restrict__ blocks, int pb, const float* __restrict__ orig,
                                 int c, int h, int w, const sige_scatter_entry* __restrict__ map,
                                 int bps, const int32_t* __restrict__ cidx, int ccount, int win,
                                 int stride, int pad, DevEpilogue epi, float* __restrict__ out) {
  long long wsz = (long long)win * win;
  long long total = (long long)ccount * c * wsz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long i = q / (c * wsz);
    int rem = static_cast<int>(q - i * c * wsz);
    int ch = rem / static_cast<int>(wsz);
    int cell = rem - ch * static_cast<int>(wsz);
    int wy = cell / win, wx = cell - wy * win;
    int n = cidx[3 * i], sy = cidx[3 * i + 1] * stride - pad + wy, sx = cidx[3 * i + 2] * stride - pad + wx;
    float v = 0.0f;
    if (sy >= 0 && sy < h && sx >= 0 && sx < w) {
      sige_scatter_entry e = map[(size_t)sy * w + sx];
      v = e.block < 0 ? __ldg(orig + (((size_t)n * c + ch) * h + sy) * w + sx)
                      : __ldg(blocks + (((size_t)(n * bps + e.block) * c + ch) * pb + e.dy) * pb + e.dx);
      v = dev_epi(epi, v, ch, c, n);
    }
    out[q] = v;
  }
}

// Residual join passes (kernels.cpp:306-334): main tiles out = m + sc_orig;
// shortcut tiles out = out + (s - sc_orig).
__global__ void k_residual(const float* __restrict__ blocks, int count, int c, int b,
                           const int32_t* __restrict__ idx, const float* __restrict__ orig_sc,
                           float* __restrict__ out, int nsamp, int h, int w, int shortcut_pass) {
  long long bsz = (long long)b * b;
  long long total = (long long)count * c * bsz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long i = q / (c * bsz);
    int rem = static_cast<int>(q - i * c * bsz);
    int ch = rem / static_cast<int>(bsz);
    int cell = rem - ch * static_cast<int>(bsz);
    const int n = idx[3 * i], y0 = idx[3 * i + 1], x0 = idx[3 * i + 2];
    int y = y0 + cell / b, xx = x0 + cell % b;
    if (y >= h || xx >= w || n < 0 || n >= nsamp || y0 < 0 || x0 < 0) continue;  // never out of the tensor
    size_t p = (((size_t)n * c + ch) * h + y) * w + xx;
    float v = blocks[q];
    out[p] = shortcut_pass ? __fadd_rn(out[p], __fsub_rn(v, orig_sc[p])) : __fadd_rn(v, orig_sc[p]);
  }
}

// add_blocks / subtract_blocks (kernels.cpp:359-380): a + sign*b.
__global__ void k_combine(const float* __restrict__ a, const float* __restrict__ b, float sign,
                          long long n, float* __restrict__ out) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x)
    out[q] = __fadd_rn(a[q], __fmul_rn(sign, b[q]));
}

// apply_epilogue_on_blocks (kernels.cpp:382-389).
__global__ void k_epilogue_blocks(float* blocks, int count, int c, int bh,
                                  const int32_t* __restrict__ idx, DevEpilogue epi) {
  long long bsz = (long long)bh * bh;
  long long total = (long long)count * c * bsz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long i = q / (c * bsz);
    int ch = static_cast<int>((q / bsz) % c);
    blocks[q] = dev_epi(epi, blocks[q], ch, c, idx[3 * i]);
  }
}

// conv core on CUDA cores (conv.cpp:33-79): per output acc = +0; for ic,
// ky, kx (in-bounds taps): acc = acc + w*x (separate roundings unless
// math == SIGE_MATH_FP32_FMA); then + bias. `in` is (planes, ih, iw) per
// sample/block with `in_stride` floats between consecutive samples/blocks.
template <int MATH>
__global__ void k_conv_cc(const float* __restrict__ in, long long in_stride, int ci, int ih, int iw,
                          const float* __restrict__ wt, const float* __restrict__ bias, int co,
                          int k, int s, int pad, float* __restrict__ out, long long out_stride,
                          int oh, int ow, int items) {
  long long per = (long long)co * oh * ow;
  long long total = per * items;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long it = q / per;
    int rem = static_cast<int>(q - it * per);
    int oc = rem / (oh * ow);
    int cell = rem - oc * oh * ow;
    int oy = cell / ow, ox = cell - oy * ow;
    const float* src = in + it * in_stride;
    const float* wk = wt + (size_t)oc * ci * k * k;
    float acc = 0.0f;
    for (int ic = 0; ic < ci; ++ic) {
      const float* plane = src + (size_t)ic * ih * iw;
      for (int ky = 0; ky < k; ++ky) {
        int iy = oy * s + ky - pad;
        if (iy < 0 || iy >= ih) continue;
        for (int kx = 0; kx < k; ++kx) {
          int ix = ox * s + kx - pad;
          if (ix < 0 || ix >= iw) continue;
          float wv = __ldg(wk + (ic * k + ky) * k + kx), xv = __ldg(plane + (size_t)iy * iw + ix);
          if (MATH == SIGE_MATH_FP32_FMA)
            acc = __fmaf_rn(wv, xv, acc);
          else
            acc = __fadd_rn(acc, __fmul_rn(wv, xv));
        }
      }
    }
    if (bias) acc = __fadd_rn(acc, __ldg(bias + oc));
    out[it * out_stride + rem] = acc;
  }
}

}  // namespace

// ------------------------------------------------------------ host side --

void op_difference_mask(const float* o, const float* e, int n, int c, int h, int w, float thr,
                        uint8_t* mask, cudaStream_t st) {
  if (thr < 0.0f) throw ConfigError("compute_difference_mask: threshold must be >= 0");
  if (n < 1 || c < 1 || h < 1 || w < 1)
    throw ConfigError("compute_difference_mask: all dims must be >= 1");
  long long hw = (long long)h * w;
  SIGE_CUDA(cudaMemsetAsync(mask, 0, hw, st));
  int planes = n * c;
  const bool vec = (hw & 3) == 0 && ((reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(e)) & 15) == 0;
  long long nq = vec ? hw / 4 : hw;
  int gx = static_cast<int>(std::min<long long>((nq + 255) / 256, 1 << 16));
  // enough CTAs for ~4 waves: split the planes across grid.y
  int want_y = std::max(1, (sm_count() * 8) / std::max(1, gx));
  int gy = std::min(planes, want_y);
  int ppy = (planes + gy - 1) / gy;
  gy = (planes + ppy - 1) / ppy;
  k_difference_mask<<<dim3(gx, gy), 256, 0, st>>>(o, e, planes, ppy, hw, thr, mask);
  after_launch("k_difference_mask");
}

void op_downsample_mask(const uint8_t* m, int h, int w, int oh, int ow, uint8_t* out,
                        cudaStream_t st) {
  if (oh < 1 || ow < 1 || oh > h || ow > w)
    throw ConfigError("downsample_mask: target must be >= 1 and <= source");
  if (h % oh != 0 || w % ow != 0)
    throw ConfigError("downsample_mask: non-integer scale factor (" + std::to_string(h) + "x" +
                      std::to_string(w) + " -> " + std::to_string(oh) + "x" +
                      std::to_string(ow) + ")");
  k_downsample_mask<<<grid_for((long long)oh * ow), kThreads, 0, st>>>(m, h, w, oh, ow, out);
  after_launch("k_downsample_mask");
}

void op_dilate_mask(const uint8_t* m, int h, int w, int r, uint8_t* out, uint8_t* tmp,
                    cudaStream_t st) {
  if (r < 0) throw ConfigError("dilate_mask: radius must be >= 0");
  if (r == 0) {
    SIGE_CUDA(cudaMemcpyAsync(out, m, (size_t)h * w, cudaMemcpyDeviceToDevice, st));
    return;
  }
  k_dilate_rows<<<grid_for((long long)h * w), kThreads, 0, st>>>(m, h, w, r, tmp);
  after_launch("k_dilate_rows");
  k_dilate_cols<<<grid_for((long long)h * w), kThreads, 0, st>>>(tmp, h, w, r, out);
  after_launch("k_dilate_cols");
}

void op_mask_to_block_indices(const uint8_t* m, int h, int w, int b, int batch, int32_t* idx,
                              int capacity, int32_t* count, cudaStream_t st) {
  if (b < 1) throw ConfigError("mask_to_block_indices: block size must be >= 1");
  if (batch < 1) throw ConfigError("mask_to_block_indices: batch must be >= 1");
  k_blockify<<<1, 1024, 0, st>>>(m, h, w, b, batch, idx, capacity, count);
  after_launch("k_blockify");
}

void op_gather(const float* x, int n, int c, int h, int w, const int32_t* idx, int count, int b,
               int ih, int iw, int k, int s, const DevEpilogue& epi, float* out, cudaStream_t st) {
  if (k != 1 && k != 3) throw ConfigError("gather: kernel size must be 1 or 3");
  if (s != 1 && s != 2) throw ConfigError("gather: stride must be 1 or 2");
  int oh = conv_out_dim(h, k, s), ow = conv_out_dim(w, k, s);
  if (ih != oh || iw != ow)
    throw ConfigError("gather: index set lives at " + std::to_string(ih) + "x" + std::to_string(iw) +
                      " but conv output of (" + std::to_string(n) + ", " + std::to_string(c) + ", " +
                      std::to_string(h) + ", " + std::to_string(w) + ") is " + std::to_string(oh) +
                      "x" + std::to_string(ow));
  if (count == 0) return;
  int win = s * b + k - s;
  static const bool rows_off = std::getenv("SIGE_GATHER_TILES") != nullptr;  // A/B: the per-tile walk
  static const bool v8_off = std::getenv("SIGE_GATHER_128") != nullptr;  // A/B: 16-byte loads for win 8
  // vector paths only on aligned tensors (a C-ABI caller may pass any float pointer)
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), oa = reinterpret_cast<uintptr_t>(out);
  const bool out16 = (oa & 15) == 0;
  if (!rows_off && !v8_off && win == 8 && (w & 7) == 0 && (xa & 31) == 0 && out16) {
    const long long rows = static_cast<long long>((count + 3) / 4) * c * 32;  // tile quads x channels x 4 x 8 rows
    const int grid = static_cast<int>(std::min<long long>((rows + 255) / 256, sm_count() * 16LL));
    k_gather_rows8w<<<grid, 256, 0, st>>>(x, c, h, w, idx, count, rows, s, (k - 1) / 2, epi, out);
    after_launch("k_gather_rows8w");
    return;
  }
  if (!rows_off && (w & 3) == 0 && (win == 8 || win == 4) && (xa & 15) == 0 && out16) {
    const long long rows = static_cast<long long>(count) * c * win;
    const int grid = static_cast<int>(std::min<long long>((rows + 255) / 256, sm_count() * 16LL));
    if (win == 8)
      k_gather_rows<8><<<grid, 256, 0, st>>>(x, c, h, w, idx, count, rows, s, (k - 1) / 2, epi, out);
    else
      k_gather_rows<4><<<grid, 256, 0, st>>>(x, c, h, w, idx, count, rows, s, (k - 1) / 2, epi, out);
    after_launch("k_gather_rows");
    return;
  }
  k_gather<<<std::min(count, sm_count() * 16), kThreads, 0, st>>>(x, c, h, w, idx, count, win, s, (k - 1) / 2,
                                                                 epi, out);
  after_launch("k_gather");
}

void op_scatter(const float* blocks, int count, int channels, int b, const int32_t* idx, float* base,
                int n, int c, int h, int w, bool add, cudaStream_t st) {
  if (channels != c) throw ConfigError(std::string(add ? "scatter_add" : "scatter") + ": channel mismatch");
  if (count == 0) return;
  const ChunkPlan cp = chunk_plan(c, b);
  const long long items = static_cast<long long>((count + cp.T - 1) / cp.T) * ((c + cp.cpi - 1) / cp.cpi);
  static const bool no_pipe = std::getenv("SIGE_SCATTER_NOPIPE") != nullptr;  // A/B: the single-buffered kernel
  const int bsz = b * b;
  static const int stage = [] {  // floats per buffer (A/B: SIGE_SCATTER_STAGE)
    const char* e = std::getenv("SIGE_SCATTER_STAGE");
    const int v = e ? std::atoi(e) : kPipeFloats;
    return std::max(1024, std::min(kPipeMaxFloats, v / 4 * 4));
  }();
  if (!no_pipe && bsz <= stage) {
    const int T = std::max(1, std::min({kMaxChunkTiles, kChunkCols / b, stage / bsz}));
    const int cpi = std::max(1, std::min(c, stage / (T * bsz)));
    const long long pitems = static_cast<long long>((count + T - 1) / T) * ((c + cpi - 1) / cpi);
    const size_t dyn = 2 * static_cast<size_t>(stage) * sizeof(float);
    static std::atomic<uint64_t> attr_done{0};
    if (first_on_device(attr_done))
      SIGE_CUDA(cudaFuncSetAttribute(k_scatter_pipe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(2 * kPipeMaxFloats * sizeof(float))));
    static int per_sm = [dyn] {
      int n = 0;
      SIGE_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_scatter_pipe, kThreads, dyn));
      return std::max(1, n);
    }();
    k_scatter_pipe<<<static_cast<int>(std::min<long long>(pitems, static_cast<long long>(sm_count()) * per_sm)),
                     kThreads, dyn, st>>>(blocks, count, c, b, idx, base, n, h, w, T, cpi, add ? 1 : 0, stage);
    after_launch("k_scatter_pipe");
    return;
  }
  static const bool no_pairs = std::getenv("SIGE_SCATTER_SINGLE") != nullptr;  // A/B: one column per thread
  const int pairs =
      !no_pairs && cp.staged && (b & 1) == 0 && (w & 1) == 0 && (reinterpret_cast<uintptr_t>(base) & 7) == 0 ? 2 : 0;
  k_scatter<<<static_cast<int>(std::min<long long>(items, sm_count() * 8LL)), kThreads, 0, st>>>(
      blocks, count, c, b, idx, base, n, h, w, cp.T, cp.cpi, cp.staged ? 1 : 0, add ? 1 : 0, pairs);
  after_launch("k_scatter");
}

void op_gather_spade(const float* x, const float* gamma, const float* beta, int n, int c, int h, int w,
                     const int32_t* idx, int count, int b, int ih, int iw, int k, int s, const DevEpilogue& epi,
                     int act, float* out, cudaStream_t st) {
  if (k != 1 && k != 3) throw ConfigError("gather: kernel size must be 1 or 3");
  if (s != 1 && s != 2) throw ConfigError("gather: stride must be 1 or 2");
  if (act < SIGE_ACT_NONE || act > SIGE_ACT_LEAKY_RELU) throw ConfigError("gather_spade: unknown activation");
  int oh = conv_out_dim(h, k, s), ow = conv_out_dim(w, k, s);
  if (ih != oh || iw != ow)
    throw ConfigError("gather: index set lives at " + std::to_string(ih) + "x" + std::to_string(iw) +
                      " but conv output of (" + std::to_string(n) + ", " + std::to_string(c) + ", " +
                      std::to_string(h) + ", " + std::to_string(w) + ") is " + std::to_string(oh) +
                      "x" + std::to_string(ow));
  if (count == 0) return;
  const int win = s * b + k - s;
  k_gather_spade<<<std::min(count, sm_count() * 16), kThreads, 0, st>>>(x, gamma, beta, c, h, w, idx, count, win,
                                                                       s, (k - 1) / 2, epi, act, out);
  after_launch("k_gather_spade");
}

void op_resize_nearest(const float* in, int n, int c, int h, int w, int oh, int ow, float* out, cudaStream_t st) {
  if (oh < 1 || ow < 1 || !((h % oh == 0) || (oh % h == 0)) || !((w % ow == 0) || (ow % w == 0)))
    throw ConfigError("resize_nearest: non-integer scale");
  const long long total = static_cast<long long>(n) * c * oh * ow;
  if (total == 0) return;
  k_resize_nearest<<<grid_for(total), kThreads, 0, st>>>(in, static_cast<long long>(n) * c, h, w, oh, ow, out);
  after_launch("k_resize_nearest");
}

int op_build_scatter_map(const int32_t* idx, int count, int b, int h, int w,
                         sige_scatter_entry* map, int* scratch2, cudaStream_t st) {
  k_map_fill<<<grid_for((long long)h * w), kThreads, 0, st>>>(map, (long long)h * w);
  after_launch("k_map_fill");
  if (count == 0) return 0;
  k_map_check<<<1, 256, 0, st>>>(idx, count, scratch2);
  after_launch("k_map_check");
  int host[2];
  SIGE_CUDA(cudaMemcpyAsync(host, scratch2, sizeof host, cudaMemcpyDeviceToHost, st));
  SIGE_CUDA(cudaStreamSynchronize(st));
  if (host[1]) throw ConfigError("build_scatter_map: tile pattern differs across batch");
  int per = host[0];
  k_map_tiles<<<grid_for((long long)per * b * b), kThreads, 0, st>>>(idx, per, b, h, w, map);
  after_launch("k_map_tiles");
  return per;
}

void op_scatter_gather(const float* blocks, int count, int pb, const float* orig, int n, int c,
                       int h, int w, const sige_scatter_entry* map, int bps, const int32_t* cidx,
                       int ccount, int cb, int ch, int cw, int k, int s, const DevEpilogue& epi,
                       float* out, cudaStream_t st) {
  if (bps * n != count) throw ConfigError("scatter_gather: map does not describe this block stack");
  if (ch != conv_out_dim(h, k, s) || cw != conv_out_dim(w, k, s))
    throw ConfigError("scatter_gather: consumer index resolution mismatch");
  if (ccount == 0) return;
  int win = s * cb + k - s;
  k_scatter_gather<<<grid_for((long long)ccount * c * win * win), kThreads, 0, st>>>(
      blocks, pb, orig, c, h, w, map, bps, cidx, ccount, win, s, (k - 1) / 2, epi, out);
  after_launch("k_scatter_gather");
}

void op_residual_pass(const float* blocks, int count, int c, int b, const int32_t* idx,
                      const float* orig_sc, float* out, int n, int h, int w, bool shortcut_pass,
                      cudaStream_t st) {
  if (count == 0) return;
  k_residual<<<grid_for((long long)count * c * b * b), kThreads, 0, st>>>(
      blocks, count, c, b, idx, orig_sc, out, n, h, w, shortcut_pass ? 1 : 0);
  after_launch("k_residual");
}

void op_combine(const float* a, const float* b, float sign, size_t n, float* out, cudaStream_t st) {
  if (n == 0) return;
  k_combine<<<grid_for((long long)n), kThreads, 0, st>>>(a, b, sign, (long long)n, out);
  after_launch("k_combine");
}

void op_epilogue_blocks(float* blocks, int count, int c, int bh, const int32_t* idx,
                        const DevEpilogue& epi, cudaStream_t st) {
  if (count == 0 || epi.num_steps == 0) return;
  k_epilogue_blocks<<<grid_for((long long)count * c * bh * bh), kThreads, 0, st>>>(blocks, count, c,
                                                                                  bh, idx, epi);
  after_launch("k_epilogue_blocks");
}

void op_conv_cc(const float* in, long long in_stride, int ci, int ih, int iw, const float* wt,
                const float* bias, int co, int k, int s, int pad, float* out, long long out_stride,
                int oh, int ow, int items, int math, cudaStream_t st) {
  if (items == 0) return;
  long long total = (long long)co * oh * ow * items;
  if (math == SIGE_MATH_FP32_FMA)
    k_conv_cc<SIGE_MATH_FP32_FMA><<<grid_for(total, 128), 128, 0, st>>>(
        in, in_stride, ci, ih, iw, wt, bias, co, k, s, pad, out, out_stride, oh, ow, items);
  else
    k_conv_cc<SIGE_MATH_EXACT><<<grid_for(total, 128), 128, 0, st>>>(
        in, in_stride, ci, ih, iw, wt, bias, co, k, s, pad, out, out_stride, oh, ow, items);
  after_launch("k_conv_cc");
}

// Device expf / SiLU over a contiguous range of float bit patterns (the GPU
// leg of the exhaustive libm sweep, tests/test_gpu_expf.py): out[i] =
// f(bits(first + i)) with f = glibc expf (mode 0) or the reference SiLU
// x / (1 + expf(-x)) (mode 1, eltwise.cpp:31-34) exactly as every exact-mode
// epilogue evaluates it.
__global__ void k_expf_sweep(uint32_t first, long long count, int mode, int fma, float* out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const float x = __uint_as_float(first + static_cast<uint32_t>(i));
    out[i] = mode == 0 ? glibc_expf(x, fma != 0) : dev_act(x, SIGE_ACT_SILU, fma, 0);
  }
}

void op_expf_sweep(uint32_t first, long long count, int mode, float* out, cudaStream_t st) {
  if (count <= 0) return;
  k_expf_sweep<<<grid_for(count), kThreads, 0, st>>>(first, count, mode, host_expf_is_fma() ? 1 : 0, out);
  after_launch("k_expf_sweep");
}

// ---- output_coverage (graph.cpp:1078-1129) building blocks on the device --
// footprint: the clipped tile rectangles of sample 0 (graph.cpp:1047-1060)
// OR-ed into m (h x w, zeroed by the caller); tile list + device count.
__global__ void k_cov_footprint(const int32_t* __restrict__ idx, const int32_t* __restrict__ count, int b, int h,
                                int w, uint8_t* __restrict__ m) {
  const int cnt = *count;
  const long long total = static_cast<long long>(cnt) * b * b;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int g = static_cast<int>(q / (b * b)), cell = static_cast<int>(q - static_cast<long long>(g) * b * b);
    if (idx[3 * g] != 0) continue;  // sample 0 only
    const int y = idx[3 * g + 1] + cell / b, x = idx[3 * g + 2] + cell % b;
    if (y < h && x < w) m[static_cast<size_t>(y) * w + x] = 1;
  }
}
// upsample_mask2x (graph.cpp:1068-1074)
__global__ void k_cov_up2(const uint8_t* __restrict__ m, int h, int w, uint8_t* __restrict__ out) {
  const long long total = 4LL * h * w;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int y = static_cast<int>(q / (2 * w)), x = static_cast<int>(q - static_cast<long long>(y) * 2 * w);
    out[q] = m[static_cast<size_t>(y / 2) * w + x / 2];
  }
}
// the empty-mask / dense cases (graph.cpp:1083-1085): value = any ? 1 : 0, or fill
__global__ void k_cov_final(uint8_t* m, long long n, const int32_t* __restrict__ any, int mode) {
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x) {
    if (mode == 1) m[q] = 1;             // not sparse: everything can change
    else if (!*any) m[q] = 0;            // empty mask: nothing changes
  }
}

void op_cov_footprint(const int32_t* idx, const int32_t* count, int capacity, int b, int h, int w, uint8_t* m,
                      cudaStream_t st) {
  if (capacity == 0) return;
  k_cov_footprint<<<grid_for(static_cast<long long>(capacity) * b * b), kThreads, 0, st>>>(idx, count, b, h, w, m);
  after_launch("k_cov_footprint");
}
void op_cov_up2(const uint8_t* m, int h, int w, uint8_t* out, cudaStream_t st) {
  k_cov_up2<<<grid_for(4LL * h * w), kThreads, 0, st>>>(m, h, w, out);
  after_launch("k_cov_up2");
}
void op_cov_final(uint8_t* m, long long n, const int32_t* any, int mode, cudaStream_t st) {
  k_cov_final<<<grid_for(n), kThreads, 0, st>>>(m, n, any, mode);
  after_launch("k_cov_final");
}

}  // namespace sige_b200
