// conv_tc.cu — fused gather -> implicit-GEMM conv -> scatter on the 5th-gen
// tensor cores (tcgen05.mma, FP32 accumulators in TMEM).
//
// Implicit GEMM without im2col. For a tile of bh x bw output pixels the CTA
// stages the tile's input window once in shared memory in the UMMA K-major
// "interleaved" (SWIZZLE_NONE) canonical layout: each 16-byte channel group
// (4 fp32 / 8 fp16 channels) is a run of window pixels at a 16-byte pitch
// (core matrices of 8 rows x 16 B, SBO = 128 B) and groups sit LBO bytes
// apart. Output pixel (oy, ox) owns GEMM row r = oy*P + ox (P = window
// pitch), so the A operand of tap (ky, kx) is the same buffer read from start
// row ky*P + kx — nine descriptor offsets, no duplicated data. Rows with
// ox >= bw are computed and discarded. Stride 2 splits the window into four
// phase planes (space-to-depth) so every tap is again a pure row shift.
// Several tiles share one M=128 MMA when their windows fit (b=6: two 64-row
// windows; b=4 1x1: eight 16-row windows).
//
// Operands: kind::tf32 (fp32 storage, 32 channels per 128-byte K chunk) or
// kind::f16 with fp16 operands (same 10-bit mantissa, 64 channels per chunk,
// half the bytes, twice the MMA rate). Both accumulate in FP32 in TMEM.
//
// Staging applies the source's pending element-wise chain (folded GroupNorm
// scale-shift + SiLU with the bit-exact glibc expf) to copied pixels only and
// leaves the zero fill untouched, exactly as gather() (kernels.cpp:39-86). The
// engine avoids that work on the hot path: a producer conv can also write
// act = chain(out) once per output pixel (Dst::act, fp16), and the consumer
// stages plain copies of it.
//
// Weights are packed [chunk][tap][group][n_pad][16 B] and streamed by TMA
// (cp.async.bulk.tensor.3d, one copy per ring stage covering 1, 3 or 9 taps
// of an N slice) through a 4-stage mbarrier ring. The N slice (16..128) is
// chosen on the device from the live tile count so even a layer with a
// handful of tiles fills the SMs. The epilogue reads TMEM with tcgen05.ld,
// adds the bias and writes the conv output / residual join straight into the
// destination with 16-byte stores (scatter fused, kernels.cpp:88-132, 291-337).
//
// Launch: programmatic dependent launch — setup, TMEM allocation and the first
// weight stages overlap the previous layer's tail (griddepcontrol.wait guards
// every access to data the previous kernel produced).
//
// Warp roles (320 threads): warps 0-7 stage A and run the epilogue (warp w
// reads TMEM lanes 32*(w%4), column half w/4); warp 8 allocates TMEM and
// issues tcgen05.mma (one thread); warp 9 issues the weight TMA (one thread).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>

#include "common.hpp"
#include "engine_kernels.hpp"

namespace sige_b200 {

namespace {

constexpr int kMaxNB = 4;      // B (weight) ring stages (max)
constexpr int kStageThreads = 256;
constexpr int kThreads = kStageThreads + 64;
constexpr int kMaxNTile = 128;  // TMEM columns allocated (fp32 accumulators)
constexpr int kBatch = 8;       // 16-byte groups staged per thread per batch

struct TcParams {
  Src src;
  Tiles tiles;
  Dst dst;
  const float* bias;
  int c_in, c_out, k, s, pad;
  int n_pad, nchunks, ntaps, phases;
  int P, Mt, T, win_h, win_w;
  int min_items;  // target number of work items (SM count)
  int nb;         // ring stages in use
  uint32_t lbo_a, idesc_base;
  int a_bytes, b_stage_bytes;
  int tps[4];     // taps per weight stage for n_tile = 16, 32, 64, 128
  unsigned long long* tl;  // debug timeline (SIGE_TC_TIMELINE), nullptr normally
};

// ------------------------------------------------------------- PTX ------
__device__ __forceinline__ void tl_mark(const TcParams& p, int idx) {
  if (p.tl && blockIdx.x < 8) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.tl[blockIdx.x * 32 + idx] = t;
  }
}
__device__ __forceinline__ void tl_cta(const TcParams& p, int base) {
  if (p.tl) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.tl[base + blockIdx.x] = t;
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0, spins = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    // A lost arrival must fail loudly instead of hanging the device.
    if (!done && ++spins > (1u << 24)) __trap();
  } while (!done);
}

__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                       uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// UMMA shared-memory descriptor, SWIZZLE_NONE K-major (version 1 for sm_100):
// start >> 4 in [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46), version bit 46.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

template <bool F16>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                     uint32_t accumulate) {
  if constexpr (F16) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------- staging --
// Row geometry is precomputed once per CTA: row_tab[q] packs, for GEMM-space
// row q = [phase][tile][Mt], the tile slot t and the window offset (wy, wx)
// (bit 31 = row carries window data). The item's tiles live in s_tile as
// (n, window origin y, x). A staging unit is (row q, 16-byte channel group j).
__device__ __forceinline__ int32_t row_info(const TcParams& p, int q) {
  const int tm = p.T * p.Mt;
  const int ph = q / tm;
  const int rem = q - ph * tm;
  const int t = rem / p.Mt, rr = rem - t * p.Mt;
  const int pr = rr / p.P, pc = rr - pr * p.P;
  const int wy = pr * p.s + (ph >> 1), wx = pc * p.s + (ph & 1);
  if (wy >= p.win_h || wx >= p.win_w) return 0;
  return static_cast<int32_t>(0x80000000u | (static_cast<uint32_t>(t) << 24) | (static_cast<uint32_t>(wy) << 12) |
                              static_cast<uint32_t>(wx));
}

// The pending element-wise chain over one unit's values, out of line so the
// glibc-expf body exists once in the kernel (instruction-cache footprint).
__device__ __noinline__ void epi_unit(const DevEpilogue& e, float* f, int cnt, int cc, int c, int n) {
  for (int i = 0; i < cnt; ++i) f[i] = dev_epi(e, f[i], cc + i, c, n);
}

__device__ __noinline__ void raw_unit(const Src& s, float* f, int cnt, int cc, int n, int y, int x) {
  for (int i = 0; i < cnt; ++i) f[i] = src_raw(s, n, cc + i, y, x);
}

// Fills A buffer with K chunk `ch`. Phase 1 resolves kBatch units and issues
// all their 16-byte loads (8-16 loads in flight per thread); phase 2 applies
// the epilogue, converts (tf32 round / fp16) and stores to shared memory.
// An fp16 source in F16 mode is a pure 16-byte copy.
template <bool F16>
__device__ __forceinline__ void stage_a(const TcParams& p, uint8_t* abuf, int ch, const int32_t* row_tab,
                                        const int4* s_tile) {
  constexpr int kG = F16 ? 8 : 4;  // channels per 16-byte group
  const int units = p.phases * p.T * p.Mt * 8;
  const Src& s = p.src;
  const bool half_src = F16 && s.half && s.layout == kNHWC && (s.c & 7) == 0 && s.epi.num_steps == 0;
  const bool vec = !s.half && s.layout == kNHWC && (s.c & 3) == 0;
  const int ph_h = s.h >> s.up, ph_w = s.w >> s.up;
  for (int u0 = threadIdx.x; u0 < units; u0 += kStageThreads * kBatch) {
    float4 raw[kBatch][kG / 4];
    int4 where[kBatch];  // (n, y, x, cc); n < 0 marks a zero unit
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int u = u0 + b * kStageThreads;
      where[b] = make_int4(-1, 0, 0, 0);
#pragma unroll
      for (int v = 0; v < kG / 4; ++v) raw[b][v] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (u >= units) continue;
      const int32_t info = row_tab[u >> 3];
      if (info >= 0) continue;  // padding row
      const int4 tl = s_tile[(info >> 24) & 0x7f];
      const int y = tl.y + ((info >> 12) & 0xfff), x = tl.z + (info & 0xfff);
      const int cc = ch * (8 * kG) + (u & 7) * kG;
      if (tl.x < 0 || y < 0 || y >= s.h || x < 0 || x >= s.w || cc >= p.c_in) continue;
      where[b] = make_int4(tl.x, y, x, cc);
      const size_t pix = (static_cast<size_t>(tl.x) * ph_h + (y >> s.up)) * ph_w + (x >> s.up);
      if (half_src) {
        raw[b][0] = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const __half*>(s.ptr) + pix * s.c + cc));
      } else if (vec) {
        const float4* base = reinterpret_cast<const float4*>(s.ptr + pix * s.c + cc);
#pragma unroll
        for (int v = 0; v < kG / 4; ++v)
          if (cc + 4 * v < p.c_in) raw[b][v] = __ldg(base + v);
      }
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int u = u0 + b * kStageThreads;
      if (u >= units) break;
      uint4 st;
      if (half_src) {
        st = *reinterpret_cast<const uint4*>(&raw[b][0]);  // already fp16, zero for empty units
      } else {
        float f[kG];
#pragma unroll
        for (int v = 0; v < kG / 4; ++v) {
          f[4 * v] = raw[b][v].x;
          f[4 * v + 1] = raw[b][v].y;
          f[4 * v + 2] = raw[b][v].z;
          f[4 * v + 3] = raw[b][v].w;
        }
        const int4 w4 = where[b];
        if (w4.x >= 0) {
          const int cnt = min(kG, p.c_in - w4.w);
          if (!vec) raw_unit(s, f, cnt, w4.w, w4.x, w4.y, w4.z);
          if (s.epi.num_steps) epi_unit(s.epi, f, cnt, w4.w, s.c, w4.x);
        }
        if constexpr (F16) {
          st = make_uint4(pack_h2(f[0], f[1]), pack_h2(f[2], f[3]), pack_h2(f[4], f[5]), pack_h2(f[6], f[7]));
        } else {
          st = make_uint4(__float_as_uint(tf32_rna(f[0])), __float_as_uint(tf32_rna(f[1])),
                          __float_as_uint(tf32_rna(f[2])), __float_as_uint(tf32_rna(f[3])));
        }
      }
      *reinterpret_cast<uint4*>(abuf + (u & 7) * p.lbo_a + (u >> 3) * 16) = st;
    }
  }
}

// ------------------------------------------------------------ epilogue --
__device__ __noinline__ float addend_val(const Src& a, int n, int oc, int y, int x) {
  return src_val(a, n, oc, y, x);
}

__device__ __noinline__ void act_store(const Dst& d, size_t p, int n, int oc0, const float* v, int cnt) {
  float a[8];
  for (int j = 0; j < cnt; ++j) a[j] = dev_epi(d.act_epi, v[j], oc0 + j, d.c, n);
  if (d.act_half) {
    __half* h = static_cast<__half*>(d.act) + p;
    if (cnt == 8 && (p & 7) == 0) {
      *reinterpret_cast<uint4*>(h) = make_uint4(pack_h2(a[0], a[1]), pack_h2(a[2], a[3]), pack_h2(a[4], a[5]),
                                                pack_h2(a[6], a[7]));
    } else {
      for (int j = 0; j < cnt; ++j) h[j] = __float2half_rn(a[j]);
    }
  } else {
    float* f = static_cast<float*>(d.act) + p;
    for (int j = 0; j < cnt; ++j) f[j] = a[j];
  }
}

// 8 consecutive output channels of one pixel: bias, write mode, optional act.
__device__ __forceinline__ void out8(const TcParams& p, size_t pix, int n, int y, int x, int oc0, float (&v)[8]) {
  const Dst& d = p.dst;
  const int cnt = min(8, p.c_out - oc0);
  if (cnt <= 0) return;
  if (p.bias) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j < cnt) v[j] = __fadd_rn(v[j], __ldg(p.bias + oc0 + j));
  }
  const size_t at = pix + oc0;
  const bool vec = cnt == 8 && (d.c & 3) == 0;
  float* o = d.ptr + at;
  if (d.mode == kStore && vec) {
    reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(o)[1] = make_float4(v[4], v[5], v[6], v[7]);
  } else if ((d.mode == kResMain || d.mode == kResShortcut) && vec) {
    const float4 a0 = __ldg(reinterpret_cast<const float4*>(d.aux + at));
    const float4 a1 = __ldg(reinterpret_cast<const float4*>(d.aux + at) + 1);
    const float aux[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    float r[8];
    if (d.mode == kResMain) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(v[j], aux[j]);
    } else {
      const float4 b0 = reinterpret_cast<const float4*>(o)[0], b1 = reinterpret_cast<const float4*>(o)[1];
      const float cur[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(cur[j], __fsub_rn(v[j], aux[j]));
    }
    reinterpret_cast<float4*>(o)[0] = make_float4(r[0], r[1], r[2], r[3]);
    reinterpret_cast<float4*>(o)[1] = make_float4(r[4], r[5], r[6], r[7]);
  } else {
    for (int j = 0; j < cnt; ++j) {
      switch (d.mode) {
        case kStore:
          o[j] = v[j];
          break;
        case kResMain:
          o[j] = __fadd_rn(v[j], __ldg(d.aux + at + j));
          break;
        case kResShortcut:
          o[j] = __fadd_rn(o[j], __fsub_rn(v[j], __ldg(d.aux + at + j)));
          break;
        default:
          o[j] = __fadd_rn(v[j], addend_val(d.addend, n, oc0 + j, y, x));
          break;
      }
    }
  }
  if (d.act) act_store(d, at, n, oc0, v, cnt);
}

// Runtime N tile: the largest power-of-two slice of n_pad (<= 128, >= 16,
// multiple of 16) that still yields >= min_items work items.
__device__ __forceinline__ int pick_n_tile(const TcParams& p, int items_m) {
  int nt = min(p.n_pad, kMaxNTile);
  while (nt > 16 && (nt / 2) % 16 == 0 && p.n_pad % (nt / 2) == 0 &&
         static_cast<long long>(items_m) * (p.n_pad / nt) < p.min_items)
    nt /= 2;
  return nt;
}

__device__ __forceinline__ int nt_index(int nt) { return nt <= 16 ? 0 : nt <= 32 ? 1 : nt <= 64 ? 2 : 3; }

template <bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_tc(const __grid_constant__ TcParams p, const __grid_constant__ TcMaps maps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_bfull[kMaxNB], bar_bempty[kMaxNB], bar_afull[2], bar_afree[2];
  __shared__ __align__(8) uint64_t bar_acc_full, bar_acc_empty;
  __shared__ uint32_t tmem_base;
  __shared__ int4 s_tile[16];  // item tiles: (n, window origin y, x, -); n = -1 for empty slots

  uint8_t* abuf[2] = {smem, smem + p.a_bytes};
  uint8_t* bbuf = smem + 2 * p.a_bytes;
  int32_t* row_tab = reinterpret_cast<int32_t*>(bbuf + p.nb * p.b_stage_bytes);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    tl_mark(p, 0);
    tl_cta(p, 256);
  }
  for (int q = threadIdx.x; q < p.phases * p.T * p.Mt; q += blockDim.x) row_tab[q] = row_info(p, q);

  if (threadIdx.x == 0) {
    for (int i = 0; i < p.nb; ++i) {
      mbar_init(&bar_bfull[i], 1);
      mbar_init(&bar_bempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_afull[i], kStageThreads);
      mbar_init(&bar_afree[i], 1);
    }
    mbar_init(&bar_acc_full, 1);
    mbar_init(&bar_acc_empty, kStageThreads);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(kMaxNTile)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tmem_base;
  if (threadIdx.x == 0) tl_mark(p, 1);
  // Tile lists / counts come from the IndexPlan, which finished before the
  // previous conv started; weights are static. Both are safe before the wait.
  const int count = p.tiles.count_dev ? *p.tiles.count_dev : p.tiles.count;
  const int items_m = (count + p.T - 1) / p.T;
  const int n_tile = pick_n_tile(p, items_m);
  const int n_slices = p.n_pad / n_tile;
  const int n_items = items_m * n_slices;
  const int nti = nt_index(n_tile);
  const int tps = p.tps[nti];
  const int tgroups = p.ntaps / tps;
  const uint32_t lbo_b = static_cast<uint32_t>(n_tile * 16);
  const uint32_t tap_b = static_cast<uint32_t>(n_tile * 128);  // one tap of B in smem
  const uint32_t idesc = p.idesc_base | (static_cast<uint32_t>(n_tile >> 3) << 17);
  if (threadIdx.x == 0) pdl_trigger();  // the next layer may start its own setup

  if (warp < 8) {
    // ---------------- A staging + epilogue ----------------
    pdl_wait();  // the source / destination were written by the previous kernel
    uint32_t a_iter = 0, it = 0;
    const int m = threadIdx.x & 127;  // TMEM lane = GEMM row
    const int half = warp >> 2;       // column half of the accumulator
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int mi = item / n_slices, ni = item % n_slices;
      const int g0 = mi * p.T, nt = min(p.T, count - g0);
      asm volatile("bar.sync 1, %0;" ::"n"(kStageThreads));  // previous item's s_tile readers done
      if (threadIdx.x < p.T) {
        const int t = threadIdx.x, g = g0 + t;
        s_tile[t] = t < nt ? make_int4(p.tiles.idx[3 * g], p.tiles.idx[3 * g + 1] * p.s - p.pad,
                                       p.tiles.idx[3 * g + 2] * p.s - p.pad, 0)
                           : make_int4(-1, 0, 0, 0);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kStageThreads));
      if (threadIdx.x == 0 && it == 0) tl_mark(p, 2);
      for (int ch = 0; ch < p.nchunks; ++ch, ++a_iter) {
        const int b = a_iter & 1;
        if (a_iter >= 2) mbar_wait(&bar_afree[b], ((a_iter >> 1) - 1) & 1);
        stage_a<F16>(p, abuf[b], ch, row_tab, s_tile);
        if (threadIdx.x == 0 && it == 0 && ch == 0) tl_mark(p, 3);
        fence_proxy_async();
        mbar_arrive(&bar_afull[b]);
      }
      if (threadIdx.x == 0 && it == 0) tl_mark(p, 4);
      mbar_wait(&bar_acc_full, it & 1);
      tc_fence_after();
      if (threadIdx.x == 0 && it == 0) tl_mark(p, 5);
      const int t = m / p.Mt, rr = m - t * p.Mt;
      const int oy = rr / p.P, ox = rr - oy * p.P;
      bool valid = t < nt && oy < p.tiles.bh && ox < p.tiles.bw;
      int n = 0, y = 0, x = 0;
      if (valid) {
        const int4 tl = s_tile[t];
        n = tl.x;
        y = (tl.y + p.pad) / p.s + oy;
        x = (tl.z + p.pad) / p.s + ox;
        valid = y < p.dst.h && x < p.dst.w;
      }
      const size_t pix = ((static_cast<size_t>(n) * p.dst.h + y) * p.dst.w + x) * p.dst.c;
      const int cols = n_tile / 2;
      for (int cb = half * cols; cb < (half + 1) * cols; cb += 8) {
        float v[8];
        tmem_ld8(taddr + (static_cast<uint32_t>((warp & 3) * 32) << 16) + static_cast<uint32_t>(cb), v);
        if (valid) out8(p, pix, n, y, x, ni * n_tile + cb, v);
      }
      if (threadIdx.x == 0 && it == 0) tl_mark(p, 6);
      tc_fence_before();
      mbar_arrive(&bar_acc_empty);
    }
  } else if (warp == 8) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      uint32_t a_iter = 0, b_iter = 0, it = 0;
      const uint32_t a0 = smem_u32(abuf[0]), a1 = smem_u32(abuf[1]), b0 = smem_u32(bbuf);
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
        if (it > 0) {
          mbar_wait(&bar_acc_empty, (it - 1) & 1);
          tc_fence_after();
        }
        for (int ch = 0; ch < p.nchunks; ++ch, ++a_iter) {
          const int b = a_iter & 1;
          mbar_wait(&bar_afull[b], (a_iter >> 1) & 1);
          tc_fence_after();
          if (it == 0 && ch == 0) tl_mark(p, 7);
          const uint32_t abase = b ? a1 : a0;
          for (int tg = 0; tg < tgroups; ++tg, ++b_iter) {
            const int st = b_iter % p.nb;
            mbar_wait(&bar_bfull[st], (b_iter / p.nb) & 1);
            tc_fence_after();
            if (b_iter == 0) tl_mark(p, 8);
            for (int tt = 0; tt < tps; ++tt) {
              const int tap = tg * tps + tt;
              const int ky = tap / p.k, kx = tap - ky * p.k;
              const int phase = p.s == 2 ? ((ky & 1) << 1) | (kx & 1) : 0;
              const int shift = (ky / p.s) * p.P + (kx / p.s);
              const uint32_t arow = abase + static_cast<uint32_t>((phase * p.T * p.Mt + shift) * 16);
              const uint32_t brow = b0 + static_cast<uint32_t>(st * p.b_stage_bytes) + tt * tap_b;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {  // 4 MMAs of K = 32 bytes each
                const uint64_t ad = umma_desc(arow + kk * 2 * p.lbo_a, p.lbo_a, 128);
                const uint64_t bd = umma_desc(brow + kk * 2 * lbo_b, lbo_b, 128);
                umma<F16>(taddr, ad, bd, idesc, (ch | tap | kk) != 0 ? 1u : 0u);
              }
            }
            umma_commit(&bar_bempty[st]);
          }
          umma_commit(&bar_afree[b]);
        }
        umma_commit(&bar_acc_full);
        if (it == 0) tl_mark(p, 9);
      }
    }
  } else {
    // ---------------- weight producer (TMA) ----------------
    if (lane == 0) {
      const CUtensorMap* map = &maps.m[nti];
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
      uint32_t b_iter = 0;
      const uint32_t b0 = smem_u32(bbuf);
      const uint32_t stage_bytes = static_cast<uint32_t>(tps) * tap_b;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int ni = item % n_slices;
        for (int ch = 0; ch < p.nchunks; ++ch)
          for (int tg = 0; tg < tgroups; ++tg, ++b_iter) {
            const int st = b_iter % p.nb;
            if (b_iter >= static_cast<uint32_t>(p.nb)) mbar_wait(&bar_bempty[st], ((b_iter / p.nb) - 1) & 1);
            mbar_expect_tx(&bar_bfull[st], stage_bytes);
            tma_3d(b0 + st * p.b_stage_bytes, map, 0, ni * n_tile, (ch * p.ntaps + tg * tps) * 8, &bar_bfull[st]);
            if (b_iter == 0) tl_mark(p, 10);
          }
        if (item == static_cast<int>(blockIdx.x)) tl_mark(p, 11);
      }
    }
  }
  if (threadIdx.x == 0) tl_mark(p, 12);
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(kMaxNTile)
                 : "memory");
    if (lane == 0) {
      tl_mark(p, 13);
      tl_cta(p, 512);
    }
  }
}

// Weight packing: out[chunk][tap][group j][n][e] = w[n][chunk*ck + j*gch + e][ky][kx]
// (tf32-rounded fp32 or fp16), zero for padded n / channels.
template <bool F16>
__global__ void k_pack_tc(const float* __restrict__ w, int c_out, int c_in, int k, int n_pad, int nchunks,
                          void* __restrict__ out) {
  const int ntaps = k * k;
  constexpr int kG = F16 ? 8 : 4;
  const long long total = static_cast<long long>(nchunks) * ntaps * 8 * n_pad * kG;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long r = q;
    const int e = static_cast<int>(r % kG);
    r /= kG;
    const int n = static_cast<int>(r % n_pad);
    r /= n_pad;
    const int j = static_cast<int>(r % 8);
    r /= 8;
    const int tap = static_cast<int>(r % ntaps);
    const int ch = static_cast<int>(r / ntaps);
    const int ic = ch * 8 * kG + j * kG + e;
    const float v = (n < c_out && ic < c_in) ? w[(static_cast<size_t>(n) * c_in + ic) * ntaps + tap] : 0.0f;
    if constexpr (F16)
      static_cast<__half*>(out)[q] = __float2half_rn(v);
    else
      static_cast<float*>(out)[q] = tf32_rna(v);
  }
}

int n_pad_for(int c_out) { return c_out <= 128 ? (c_out + 15) / 16 * 16 : (c_out + 127) / 128 * 128; }

// Taps per weight stage for an N slice: small slices batch more taps per TMA.
int tps_for(int n_tile, int ntaps) {
  if (ntaps == 1) return 1;
  if (n_tile <= 16) return 9;
  if (n_tile <= 64) return 3;
  return 1;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    SIGE_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

}  // namespace

void pack_weights_tc(const float* w_dev, int c_out, int c_in, int k, int f16, ConvW* cw, cudaStream_t st) {
  const int ck = f16 ? 64 : 32;
  const int esize = f16 ? 2 : 4;
  cw->n_pad = n_pad_for(c_out);
  cw->k_pad = (c_in + ck - 1) / ck * ck;
  const int nchunks = cw->k_pad / ck, ntaps = k * k;
  const size_t total = static_cast<size_t>(nchunks) * ntaps * 8 * cw->n_pad * (16 / esize);
  void* out = nullptr;
  SIGE_CUDA(cudaMalloc(&out, total * esize));
  const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((total + 255) / 256, sm_count() * 16LL)));
  if (f16)
    k_pack_tc<true><<<grid, 256, 0, st>>>(w_dev, c_out, c_in, k, cw->n_pad, nchunks, out);
  else
    k_pack_tc<false><<<grid, 256, 0, st>>>(w_dev, c_out, c_in, k, cw->n_pad, nchunks, out);
  after_launch("k_pack_tc");
  SIGE_CUDA(cudaStreamSynchronize(st));
  cw->w_tc = out;
  // One 3-D tensor map per N-slice width: dims (16-byte element group, n, (chunk, tap, group)),
  // box (group, n_tile, taps_per_stage * 8) — a ring stage is one TMA.
  const int sizes[4] = {16, 32, 64, 128};
  for (int i = 0; i < 4; ++i) {
    const int nt = std::min(sizes[i], cw->n_pad);
    const int tps = tps_for(nt, ntaps);
    cw->maps.tps[i] = tps;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(16 / esize), static_cast<cuuint64_t>(cw->n_pad),
                                static_cast<cuuint64_t>(nchunks) * ntaps * 8};
    const cuuint64_t strides[2] = {16, static_cast<cuuint64_t>(cw->n_pad) * 16};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(16 / esize), static_cast<cuuint32_t>(nt),
                               static_cast<cuuint32_t>(tps * 8)};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&cw->maps.m[i], f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                             3, out, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  }
}

void launch_conv_tc(const Src& src, const Tiles& tiles, const ConvW& cw, const Dst& dst, int f16,
                    cudaStream_t st) {
  if (!cw.w_tc) throw ConfigError("conv (tensor core): weights were not packed for this path");
  if (tiles.capacity == 0) return;
  TcParams p{};
  p.src = src;
  p.tiles = tiles;
  p.dst = dst;
  p.bias = cw.bias;
  p.c_in = cw.c_in;
  p.c_out = cw.c_out;
  p.k = cw.k;
  p.s = cw.stride;
  p.pad = (cw.k - 1) / 2;
  p.n_pad = cw.n_pad;
  p.nchunks = cw.k_pad / (f16 ? 64 : 32);
  p.ntaps = cw.k * cw.k;
  for (int i = 0; i < 4; ++i) p.tps[i] = cw.maps.tps[i];
  const int bh = tiles.bh, bw = tiles.bw;
  int rows_ph;
  if (cw.stride == 1) {
    p.phases = 1;
    p.P = bw + cw.k - 1;
    rows_ph = bh + cw.k - 1;
  } else {
    if (cw.k == 1) throw ConfigError("conv (tensor core): 1x1 stride-2 convs are not supported");
    p.phases = 4;
    p.P = bw + 1;
    rows_ph = bh + 1;
  }
  p.win_h = (bh - 1) * cw.stride + cw.k;
  p.win_w = (bw - 1) * cw.stride + cw.k;
  const int wr = rows_ph * p.P;
  const int vr = (bh - 1) * p.P + bw;  // GEMM rows that carry valid outputs
  if (wr <= 128) {
    int mt = 16;
    while (mt < wr) mt <<= 1;
    p.Mt = mt;
    p.T = 128 / mt;
  } else {
    if (vr > 128)
      throw ConfigError("conv (tensor core): tile " + std::to_string(bh) + "x" + std::to_string(bw) +
                        " does not fit one M=128 MMA");
    p.Mt = (wr + 7) / 8 * 8;
    p.T = 1;
  }
  if (p.T > 16) throw ConfigError("conv (tensor core): more than 16 tiles per MMA");
  const int pad_rows = cw.k == 3 ? (cw.stride == 1 ? 2 * p.P + 2 : p.P + 1) : 0;
  int r_total = p.phases * p.T * p.Mt + pad_rows + 8;
  r_total = (r_total + 7) / 8 * 8 + 1;  // odd number of 16-byte rows spreads groups over banks
  p.lbo_a = static_cast<uint32_t>(r_total * 16);
  p.a_bytes = (r_total * 16 * 8 + 1023) / 1024 * 1024;
  int max_stage = 0;
  const int sizes[4] = {16, 32, 64, 128};
  for (int i = 0; i < 4; ++i) max_stage = std::max(max_stage, p.tps[i] * std::min(sizes[i], p.n_pad) * 128);
  p.b_stage_bytes = (max_stage + 1023) / 1024 * 1024;
  p.min_items = sm_count();
  const uint32_t fmt = f16 ? 0u : 2u;
  p.idesc_base = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(128 >> 4) << 24);
  const size_t fixed = 2 * static_cast<size_t>(p.a_bytes) + sizeof(int32_t) * p.phases * p.T * p.Mt;
  p.nb = kMaxNB;
  while (p.nb > 2 && fixed + static_cast<size_t>(p.nb) * p.b_stage_bytes > 220 * 1024) --p.nb;
  const size_t smem = fixed + static_cast<size_t>(p.nb) * p.b_stage_bytes;
  if (smem > 220 * 1024)
    throw ConfigError("conv (tensor core): staging needs " + std::to_string(smem) + " B of shared memory");
  static std::once_flag attr_once;
  std::call_once(attr_once, [] {
    SIGE_CUDA(cudaFuncSetAttribute(k_conv_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    SIGE_CUDA(cudaFuncSetAttribute(k_conv_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  });
  static unsigned long long* tl_buf = nullptr;
  static const bool timeline = std::getenv("SIGE_TC_TIMELINE") != nullptr;
  if (timeline) {
    if (!tl_buf) SIGE_CUDA(cudaMalloc(&tl_buf, 1024 * sizeof(unsigned long long)));
    SIGE_CUDA(cudaMemsetAsync(tl_buf, 0, 1024 * sizeof(unsigned long long), st));
    p.tl = tl_buf;
  }
  const long long max_items = static_cast<long long>((tiles.capacity + p.T - 1) / p.T) * (p.n_pad / 16);
  const int grid = static_cast<int>(std::max(1LL, std::min<long long>(max_items, sm_count())));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (f16)
    SIGE_CUDA(cudaLaunchKernelEx(&cfg, k_conv_tc<true>, p, cw.maps));
  else
    SIGE_CUDA(cudaLaunchKernelEx(&cfg, k_conv_tc<false>, p, cw.maps));
  after_launch("k_conv_tc");
  if (timeline) {
    unsigned long long h[1024];
    SIGE_CUDA(cudaMemcpyAsync(h, tl_buf, sizeof h, cudaMemcpyDeviceToHost, st));
    SIGE_CUDA(cudaStreamSynchronize(st));
    unsigned long long t0 = ~0ull, tend = 0, last = 0;
    for (int i = 0; i < grid; ++i)
      if (h[256 + i]) {
        t0 = std::min(t0, h[256 + i]);
        tend = std::max(tend, h[512 + i]);
      }
    for (int i = 0; i < grid; ++i)
      if (h[256 + i]) last = std::max(last, h[256 + i] - t0);
    std::fprintf(stderr, "[tc] %dx%d c%d->%d k%d s%d T%d Mt%d grid %d nb %d: span %.2f us, last entry %.2f us\n",
                 tiles.bh, tiles.bw, cw.c_in, cw.c_out, cw.k, cw.stride, p.T, p.Mt, grid, p.nb, (tend - t0) * 1e-3,
                 last * 1e-3);
    for (int c = 0; c < 2; ++c) {
      std::fprintf(stderr, "  cta%d:", c);
      for (int e = 0; e < 14; ++e)
        std::fprintf(stderr, " %d:%.2f", e, h[c * 32 + e] ? (h[c * 32 + e] - t0) * 1e-3 : -1.0);
      std::fprintf(stderr, "\n");
    }
  }
}

}  // namespace sige_b200
