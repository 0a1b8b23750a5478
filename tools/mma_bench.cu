// mma_bench.cu — microbenchmark of tcgen05.mma issue/complete rate on one SM
// (developer tool, not part of the library): cycles per MMA for
// kind::tf32 / kind::f16, N = 16..256, SWIZZLE_NONE (interleaved) vs
// SWIZZLE_128B K-major operands, one accumulator vs several rotating ones.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench tools/mma_bench.cu && ./mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | ((uint64_t)layout << 61);
}

template <bool F16>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (F16)
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
  return pred != 0;
}

template <bool F16>
__global__ void k_bench(int n, int layout, int naccs, int reps, int warp_issue, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp_issue == 1 || warp_issue == 3 ? threadIdx.x < 32 : threadIdx.x == 0) {
    const uint32_t a0 = su32(sm), b0 = su32(sm + 64 * 1024);
    const uint32_t fmt = F16 ? 0u : 2u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t phase = 0;
    long long best = 1ll << 60;
    for (int trial = 0; trial < 3; ++trial) {
      long long t0 = clock64();
      if (warp_issue == 3) {
        // converged warp, per-MMA descriptors = base + (tap, kk) offsets, elect per MMA
        const uint64_t ad0 = desc(a0, 2576, 128, 0), bd0 = desc(b0, n * 16, 128, 0);
        const int P = 8 + (n & 1);  // runtime-ish
        for (int r = 0; r < reps; r += 36) {
#pragma unroll
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t shift = (uint32_t)((tap / 3) * P + (tap % 3));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint64_t ad = ad0 + shift + (uint32_t)(kk * 2 * 2576 / 16);
              const uint64_t bd = bd0 + (uint32_t)(kk * 2 * n);
              if (elect_one()) mma<F16>(tbase, ad, bd, idesc, (r | tap | kk) ? 1u : 0u);
            }
          }
        }
      } else if (warp_issue == 2) {
        // loop-invariant descriptors, unrolled issue
        const uint64_t ad = layout == 0 ? desc(a0, 2576, 128, 0) : desc(a0, 16, 1024, 2);
        const uint64_t bd = layout == 0 ? desc(b0, n * 16, 128, 0) : desc(b0, 16, 1024, 2);
        const uint32_t d = tbase;
#pragma unroll 16
        for (int r = 0; r < reps; ++r) mma<F16>(d, ad, bd, idesc, r > 0 ? 1u : 0u);
      } else
      for (int r = 0; r < reps; ++r) {
        const int kk = r & 3;
        uint64_t ad, bd;
        if (layout == 0) {  // interleaved: K core matrices LBO apart
          ad = desc(a0 + kk * 2 * 2576, 2576, 128, 0);
          bd = desc(b0 + kk * 2 * n * 16, n * 16, 128, 0);
        } else {            // 128B swizzle K-major: rows of 128 B, 8-row atoms 1024 B
          ad = desc(a0 + kk * 32, 16, 1024, 2);
          bd = desc(b0 + kk * 32, 16, 1024, 2);
        }
        const uint32_t d = tbase + (uint32_t)((r % naccs) * 128);
        if (warp_issue != 1 || elect_one()) mma<F16>(d, ad, bd, idesc, r >= naccs ? 1u : 0u);
        if (warp_issue == 1) __syncwarp();
      }
      if ((warp_issue != 1 && warp_issue != 3) || elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      uint32_t done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(su32(&bar)), "r"(phase) : "memory");
      phase ^= 1;
      long long t1 = clock64();
      if (t1 - t0 < best) best = t1 - t0;
    }
    if (threadIdx.x == 0) *out = best;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k_bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(k_bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int reps = 252;
  printf("warp kind  layout  N    accs  cyc/MMA  MAC/cyc\n");
  for (int wi = 2; wi < 4; ++wi)
  for (int f16 = 0; f16 < 2; ++f16)
    for (int layout = 0; layout < 2; ++layout)
      for (int n : {16, 32, 64, 128, 256})
        for (int naccs : {1, 2}) {
          if (n * naccs > 512) continue;
          if (naccs > 1 && n > 128) continue;
          if (f16) k_bench<true><<<1, 128, 160 * 1024>>>(n, layout, naccs, reps, wi, d);
          else k_bench<false><<<1, 128, 160 * 1024>>>(n, layout, naccs, reps, wi, d);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
          long long c;
          cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
          double per = (double)c / reps;
          double macs = 128.0 * n * (f16 ? 16 : 8);
          printf("%-4d %-5s %-7s %-4d %-5d %8.1f %8.0f\n", wi, f16 ? "f16" : "tf32", layout ? "sw128" : "none", n, naccs, per, macs / per);
        }
  return 0;
}
