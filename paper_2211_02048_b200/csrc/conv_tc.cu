// conv_tc.cu — fused gather -> implicit-GEMM conv -> scatter on the 5th-gen
// tensor cores (tcgen05.mma kind::tf32, FP32 accumulators in TMEM).
//
// Implicit GEMM without im2col. For a tile of bh x bw output pixels the CTA
// stages the tile's input window once in shared memory as the UMMA K-major
// "interleaved" (SWIZZLE_NONE) canonical layout: each 4-channel group is a
// run of window pixels at a 16-byte pitch (core matrices of 8 rows x 16 B,
// SBO = 128 B) and groups sit LBO bytes apart. Output pixel (oy, ox) owns GEMM
// row r = oy*P + ox (P = window pitch), so the A operand of tap (ky, kx) is
// the same buffer read from start row (ky*P + kx) — nine descriptor offsets,
// no duplicated data. Rows with ox >= bw are computed and discarded. Stride 2
// splits the window into four phase planes (space-to-depth) so each tap is
// again a pure row shift. Several tiles share one M=128 MMA when their
// windows fit (b=6: two 64-row windows; b=4 1x1: eight 16-row windows).
//
// The staging pass applies the source's pending element-wise chain (folded
// GroupNorm scale-shift + SiLU with the bit-exact glibc expf) to copied pixels
// only and leaves the zero fill untouched, exactly as gather()
// (proj/src/kernels.cpp:39-86). Weights are pre-packed per (N tile, 32-channel
// chunk, tap) in the B-operand layout and streamed by cp.async.bulk (TMA bulk
// copy) through a 4-stage mbarrier ring. The epilogue reads TMEM with
// tcgen05.ld, adds the bias and writes the conv output / residual join
// straight into the destination (scatter fused, kernels.cpp:88-132, 291-337).
//
// Warp roles (192 threads): warps 0-3 stage A and run the epilogue (TMEM
// lanes 0-127), warp 4 allocates TMEM and issues tcgen05.mma (one thread),
// warp 5 issues the weight bulk copies (one thread).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "common.hpp"
#include "engine_kernels.hpp"

namespace sige_b200 {

namespace {

constexpr int kNB = 4;        // B (weight) ring stages
constexpr int kCK = 32;       // channels per K chunk (8 groups of 4 = 128 B per pixel row)
constexpr int kThreads = 192;

struct TcParams {
  Src src;
  Tiles tiles;
  Dst dst;
  const float* wtc;
  const float* bias;
  int c_in, c_out, k, s, pad;
  int n_tile, n_tiles_n, nchunks, ntaps, phases;
  int P, Mt, T, win_h, win_w;
  uint32_t lbo_a, lbo_b, idesc;
  int a_bytes, b_bytes, tmem_cols;
};

// ------------------------------------------------------------- PTX ------
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
  uint32_t done = 0;
  uint32_t spins = 0;
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

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
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

// UMMA shared-memory descriptor, SWIZZLE_NONE K-major (version 1 for sm_100):
// start >> 4 in [0,14), LBO >> 4 in [16,30), SBO >> 4 in [32,46), version bit 46.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ------------------------------------------------------------- staging --
// Fills A buffer `abuf` with K chunk `ch` of the windows of tiles g0..g0+nt-1:
// rows [phase][tile][Mt], channel groups LBO apart, values after the pending
// epilogue, rounded to TF32; cells outside the canvas are +0 (never epilogued).
__device__ __forceinline__ void stage_a(const TcParams& p, uint8_t* abuf, int ch, int g0, int nt,
                                        int count) {
  const int rows = p.phases * p.T * p.Mt;
  const int c0 = ch * kCK;
  for (int e = threadIdx.x; e < rows * 8; e += 128) {
    const int j = e & 7, q = e >> 3;
    const int ph = q / (p.T * p.Mt);
    const int rem = q - ph * (p.T * p.Mt);
    const int t = rem / p.Mt, rr = rem - t * p.Mt;
    const int pr = rr / p.P, pc = rr - pr * p.P;
    const int wy = pr * p.s + (ph >> 1), wx = pc * p.s + (ph & 1);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int g = g0 + t;
    if (t < nt && g < count && wy < p.win_h && wx < p.win_w) {
      const int n = p.tiles.idx[3 * g];
      const int y = p.tiles.idx[3 * g + 1] * p.s - p.pad + wy;
      const int x = p.tiles.idx[3 * g + 2] * p.s - p.pad + wx;
      const int cc = c0 + 4 * j;
      if (y >= 0 && y < p.src.h && x >= 0 && x < p.src.w && cc < p.c_in) {
        const Src& s = p.src;
        float f[4];
        if (s.layout == kNHWC && (s.c & 3) == 0) {
          const int ph_h = s.h >> s.up, ph_w = s.w >> s.up;
          const float4 raw = __ldg(reinterpret_cast<const float4*>(
              s.ptr + ((static_cast<size_t>(n) * ph_h + (y >> s.up)) * ph_w + (x >> s.up)) * s.c + cc));
          f[0] = raw.x;
          f[1] = raw.y;
          f[2] = raw.z;
          f[3] = raw.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) f[u] = cc + u < p.c_in ? src_raw(s, n, cc + u, y, x) : 0.0f;
        }
        if (s.epi.num_steps) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (cc + u < p.c_in) f[u] = dev_epi(s.epi, f[u], cc + u, s.c, n);
        }
        v = make_float4(tf32_rna(f[0]), tf32_rna(f[1]), tf32_rna(f[2]), tf32_rna(f[3]));
      }
    }
    *reinterpret_cast<float4*>(abuf + j * p.lbo_a + q * 16) = v;
  }
}

// ------------------------------------------------------------ epilogue --
__device__ __forceinline__ void out_write(const Dst& d, size_t p, int oc, int n, int y, int x, float v) {
  switch (d.mode) {
    case kStore:
      d.ptr[p] = v;
      break;
    case kResMain:
      d.ptr[p] = __fadd_rn(v, __ldg(d.aux + p));
      break;
    case kResShortcut:
      d.ptr[p] = __fadd_rn(d.ptr[p], __fsub_rn(v, __ldg(d.aux + p)));
      break;
    default:
      d.ptr[p] = __fadd_rn(v, src_val(d.addend, n, oc, y, x));
      break;
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_conv_tc(const TcParams p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t bar_bfull[kNB], bar_bempty[kNB], bar_afull[2], bar_afree[2];
  __shared__ __align__(8) uint64_t bar_acc_full, bar_acc_empty;
  __shared__ uint32_t tmem_base;

  uint8_t* abuf[2] = {smem, smem + p.a_bytes};
  uint8_t* bbuf = smem + 2 * p.a_bytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNB; ++i) {
      mbar_init(&bar_bfull[i], 1);
      mbar_init(&bar_bempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_afull[i], 128);
      mbar_init(&bar_afree[i], 1);
    }
    mbar_init(&bar_acc_full, 1);
    mbar_init(&bar_acc_empty, 128);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t taddr = tmem_base;

  const int count = p.tiles.count_dev ? *p.tiles.count_dev : p.tiles.count;
  const int items_m = (count + p.T - 1) / p.T;
  const int n_items = items_m * p.n_tiles_n;

  if (warp < 4) {
    // ---------------- A staging + epilogue ----------------
    uint32_t a_iter = 0, it = 0;
    const int m = threadIdx.x;  // TMEM lane = GEMM row
    for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++it) {
      const int mi = item / p.n_tiles_n, ni = item % p.n_tiles_n;
      const int g0 = mi * p.T, nt = min(p.T, count - g0);
      for (int ch = 0; ch < p.nchunks; ++ch, ++a_iter) {
        const int b = a_iter & 1;
        if (a_iter >= 2) mbar_wait(&bar_afree[b], ((a_iter >> 1) - 1) & 1);
        stage_a(p, abuf[b], ch, g0, nt, count);
        fence_proxy_async();
        mbar_arrive(&bar_afull[b]);
      }
      // epilogue: row m -> (tile t, output pixel)
      mbar_wait(&bar_acc_full, it & 1);
      tc_fence_after();
      const int t = m / p.Mt, rr = m - t * p.Mt;
      const int oy = rr / p.P, ox = rr - oy * p.P;
      bool valid = t < nt && oy < p.tiles.bh && ox < p.tiles.bw && (p.T > 1 || m < p.Mt);
      int n = 0, y = 0, x = 0;
      if (valid) {
        const int g = g0 + t;
        n = p.tiles.idx[3 * g];
        y = p.tiles.idx[3 * g + 1] + oy;
        x = p.tiles.idx[3 * g + 2] + ox;
        valid = y < p.dst.h && x < p.dst.w;
      }
      const size_t pix = ((static_cast<size_t>(n) * p.dst.h + y) * p.dst.w + x) * p.dst.c;
      for (int cb = 0; cb < p.n_tile; cb += 32) {
        float v[32];
        tmem_ld32(taddr + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(cb), v);
        if (!valid) continue;
        const int oc0 = ni * p.n_tile + cb;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int oc = oc0 + j;
          if (oc < p.c_out) {
            const float val = p.bias ? __fadd_rn(v[j], __ldg(p.bias + oc)) : v[j];
            out_write(p.dst, pix + oc, oc, n, y, x, val);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bar_acc_empty);
    }
  } else if (warp == 4) {
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
          const uint32_t abase = b ? a1 : a0;
          for (int tap = 0; tap < p.ntaps; ++tap, ++b_iter) {
            const int st = b_iter % kNB;
            mbar_wait(&bar_bfull[st], (b_iter / kNB) & 1);
            tc_fence_after();
            const int ky = tap / p.k, kx = tap - ky * p.k;
            const int phase = p.s == 2 ? ((ky & 1) << 1) | (kx & 1) : 0;
            const int shift = (ky / p.s) * p.P + (kx / p.s);
            const uint32_t arow = abase + static_cast<uint32_t>((phase * p.T * p.Mt + shift) * 16);
            const uint32_t brow = b0 + static_cast<uint32_t>(st * p.b_bytes);
#pragma unroll
            for (int kk = 0; kk < kCK / 8; ++kk) {
              const uint64_t ad = umma_desc(arow + kk * 2 * p.lbo_a, p.lbo_a, 128);
              const uint64_t bd = umma_desc(brow + kk * 2 * p.lbo_b, p.lbo_b, 128);
              umma_tf32(taddr, ad, bd, p.idesc, (ch | tap | kk) != 0 ? 1u : 0u);
            }
            umma_commit(&bar_bempty[st]);
          }
          umma_commit(&bar_afree[b]);
        }
        umma_commit(&bar_acc_full);
      }
    }
  } else {
    // ---------------- weight producer ----------------
    if (lane == 0) {
      uint32_t b_iter = 0;
      const size_t blk = static_cast<size_t>(p.n_tile) * kCK;  // floats per (chunk, tap) block
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int ni = item % p.n_tiles_n;
        for (int ch = 0; ch < p.nchunks; ++ch)
          for (int tap = 0; tap < p.ntaps; ++tap, ++b_iter) {
            const int st = b_iter % kNB;
            if (b_iter >= kNB) mbar_wait(&bar_bempty[st], ((b_iter / kNB) - 1) & 1);
            mbar_expect_tx(&bar_bfull[st], p.b_bytes);
            const float* src = p.wtc + ((static_cast<size_t>(ni) * p.nchunks + ch) * p.ntaps + tap) * blk;
            bulk_g2s(bbuf + st * p.b_bytes, src, p.b_bytes, &bar_bfull[st]);
          }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(p.tmem_cols)
                 : "memory");
  }
}

// Weight packing: W_tc[nt][chunk][tap][group j][n][4] = tf32(w[n][chunk*32+4j+e][ky][kx]).
__global__ void k_pack_tc(const float* __restrict__ w, int c_out, int c_in, int k, int n_tile,
                          int n_tiles_n, int nchunks, float* __restrict__ out) {
  const int ntaps = k * k;
  const long long total = static_cast<long long>(n_tiles_n) * nchunks * ntaps * 8 * n_tile * 4;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    long long r = q;
    const int e = static_cast<int>(r % 4);
    r /= 4;
    const int nl = static_cast<int>(r % n_tile);
    r /= n_tile;
    const int j = static_cast<int>(r % 8);
    r /= 8;
    const int tap = static_cast<int>(r % ntaps);
    r /= ntaps;
    const int ch = static_cast<int>(r % nchunks);
    const int nt = static_cast<int>(r / nchunks);
    const int oc = nt * n_tile + nl, ic = ch * kCK + 4 * j + e;
    float v = 0.0f;
    if (oc < c_out && ic < c_in) v = w[(static_cast<size_t>(oc) * c_in + ic) * ntaps + tap];
    out[q] = tf32_rna(v);
  }
}

int n_pad_for(int c_out) { return c_out <= 128 ? (c_out + 15) / 16 * 16 : (c_out + 127) / 128 * 128; }
int n_tile_for(int n_pad) { return std::min(n_pad, 128); }

}  // namespace

float* pack_weights_tc(const float* w_dev, int c_out, int c_in, int k, int* n_pad, int* k_pad,
                       cudaStream_t st) {
  *n_pad = n_pad_for(c_out);
  *k_pad = (c_in + kCK - 1) / kCK * kCK;
  const int n_tile = n_tile_for(*n_pad), n_tiles_n = *n_pad / n_tile, nchunks = *k_pad / kCK;
  const size_t total = static_cast<size_t>(n_tiles_n) * nchunks * k * k * n_tile * kCK;
  float* out = nullptr;
  SIGE_CUDA(cudaMalloc(&out, total * sizeof(float)));
  k_pack_tc<<<std::max<long long>(1, std::min<long long>((total + 255) / 256, sm_count() * 16LL)), 256, 0, st>>>(
      w_dev, c_out, c_in, k, n_tile, n_tiles_n, nchunks, out);
  after_launch("k_pack_tc");
  SIGE_CUDA(cudaStreamSynchronize(st));
  return out;
}

void launch_conv_tc(const Src& src, const Tiles& tiles, const ConvW& cw, const Dst& dst,
                    cudaStream_t st) {
  if (!cw.w_tc) throw ConfigError("conv (tf32): weights were not packed for the tensor-core path");
  if (tiles.capacity == 0) return;
  TcParams p{};
  p.src = src;
  p.tiles = tiles;
  p.dst = dst;
  p.wtc = cw.w_tc;
  p.bias = cw.bias;
  p.c_in = cw.c_in;
  p.c_out = cw.c_out;
  p.k = cw.k;
  p.s = cw.stride;
  p.pad = (cw.k - 1) / 2;
  p.n_tile = n_tile_for(cw.n_pad);
  p.n_tiles_n = cw.n_pad / p.n_tile;
  p.nchunks = cw.k_pad / kCK;
  p.ntaps = cw.k * cw.k;
  // Window geometry: P = window pitch per phase plane, rows per phase.
  const int bh = tiles.bh, bw = tiles.bw;
  int rows_ph;
  if (cw.stride == 1) {
    p.phases = 1;
    p.P = bw + cw.k - 1;
    rows_ph = bh + cw.k - 1;
  } else {
    if (cw.k == 1) throw ConfigError("conv (tf32): 1x1 stride-2 convs are not supported");
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
      throw ConfigError("conv (tf32): tile " + std::to_string(bh) + "x" + std::to_string(bw) +
                        " does not fit one M=128 MMA");
    p.Mt = (wr + 7) / 8 * 8;
    p.T = 1;
  }
  const int pad_rows = cw.k == 3 ? (cw.stride == 1 ? 2 * p.P + 2 : p.P + 1) : 0;
  int r_total = p.phases * p.T * p.Mt + pad_rows + 8;
  r_total = (r_total + 7) / 8 * 8 + 1;  // odd number of 16-byte rows spreads groups over banks
  p.lbo_a = static_cast<uint32_t>(r_total * 16);
  p.a_bytes = (r_total * 16 * 8 + 1023) / 1024 * 1024;
  p.lbo_b = static_cast<uint32_t>(p.n_tile * 16);
  p.b_bytes = p.n_tile * kCK * 4;
  p.tmem_cols = 32;
  while (p.tmem_cols < p.n_tile) p.tmem_cols <<= 1;
  // idesc (kind::tf32): D f32 [4,6)=1, A tf32 [7,10)=2, B tf32 [10,13)=2,
  // K-major A/B, N>>3 at [17,23), M>>4 at [24,29).
  p.idesc = (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(p.n_tile >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  const size_t smem = 2 * static_cast<size_t>(p.a_bytes) + static_cast<size_t>(kNB) * p.b_bytes;
  if (smem > 220 * 1024)
    throw ConfigError("conv (tf32): staging needs " + std::to_string(smem) + " B of shared memory");
  static size_t configured = 0;
  if (smem > configured) {
    SIGE_CUDA(cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    configured = 220 * 1024;
  }
  const long long items = static_cast<long long>((tiles.capacity + p.T - 1) / p.T) * p.n_tiles_n;
  const int grid = static_cast<int>(std::max(1LL, std::min<long long>(items, sm_count())));
  k_conv_tc<<<grid, kThreads, smem, st>>>(p);
  after_launch("k_conv_tc");
}

}  // namespace sige_b200
