// sw128_probe.cu — developer probe (not part of the library): does a
// tcgen05.mma K-major SWIZZLE_128B A descriptor that starts r rows (r*128 B)
// into a TMA-written 128B-swizzled tile read the rows r.. correctly when the
// descriptor's base-offset field carries (start >> 7) & 7?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o sw128_probe tools/sw128_probe.cu -lcuda && ./sw128_probe
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, int base_off_mode) {
  // start >> 4 [0,14), LBO >> 4 = 1 [16,30), SBO = 1024 >> 4 [32,46), version 1 at 46,
  // base offset [49,52), layout SWIZZLE_128B = 2 at [61,64)
  uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
               (2ull << 61);
  if (base_off_mode == 1) d |= (uint64_t)((addr >> 7) & 7) << 49;
  return d;
}

// A: 256 rows x 64 fp16 (K) via TMA SW128 into smem; B: 64 (N) x 64 fp16 rows via TMA SW128.
// D[m][n] = sum_k A[m + shift][k] * B[n][k], M = 128, N = 64, K = 64 (4 MMAs of K=16).
__global__ void k_probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, int shift,
                        int mode, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar, mbar;
  __shared__ uint32_t tbase;
  uint8_t* a = sm;              // 256 rows x 128 B = 32 KB
  uint8_t* b = sm + 32 * 1024;  // 64 rows x 128 B = 8 KB
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(40 * 1024) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(a)),
        "l"(&ma), "r"(0), "r"(0), "r"(su32(&bar))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(b)),
        "l"(&mb), "r"(0), "r"(0), "r"(su32(&bar))
        : "memory");
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((128u >> 4) << 24);  // f16 in, f32 acc, N=64, M=128
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = desc_sw128(su32(a) + shift * 128 + kk * 32, mode);
      const uint64_t bd = desc_sw128(su32(b) + kk * 32, mode);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                       tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(kk ? 1u : 0u)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mbar)) : "memory");
    done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(su32(&mbar)) : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // 4 warps x 32 lanes = 128 rows, 64 columns each
  const int row = threadIdx.x;
  for (int c0 = 0; c0 < 64; c0 += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tbase + ((uint32_t)((threadIdx.x / 32) * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) out[row * 64 + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase) : "memory");
}

int main() {
  const int RA = 256, K = 64, N = 64;
  std::vector<__half> ha(RA * K), hb(N * K);
  std::vector<float> fa(RA * K), fb(N * K);
  srand(1);
  for (int i = 0; i < RA * K; ++i) {
    fa[i] = (float)(rand() % 7 - 3);
    ha[i] = __float2half(fa[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    fb[i] = (float)(rand() % 5 - 2);
    hb[i] = __float2half(fb[i]);
  }
  __half *da, *db;
  float* dout;
  cudaMalloc(&da, RA * K * 2);
  cudaMalloc(&db, N * K * 2);
  cudaMalloc(&dout, 128 * 64 * 4);
  cudaMemcpy(da, ha.data(), RA * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (CUresult(*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill))fnp;
  CUtensorMap ma, mb;
  cuuint64_t dimA[2] = {(cuuint64_t)K, (cuuint64_t)RA}, strA[1] = {(cuuint64_t)K * 2};
  cuuint32_t boxA[2] = {64, 256}, es[2] = {1, 1};
  cuuint64_t dimB[2] = {(cuuint64_t)K, (cuuint64_t)N}, strB[1] = {(cuuint64_t)K * 2};
  cuuint32_t boxB[2] = {64, 64};
  CUresult r1 = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, da, dimA, strA, boxA, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, db, dimB, strB, boxB, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  std::vector<float> got(128 * 64);
  for (int mode = 0; mode < 2; ++mode)
    for (int shift : {0, 1, 3, 7, 8, 9, 21, 38}) {
      k_probe<<<1, 128, 48 * 1024>>>(ma, mb, shift, mode, dout);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("mode %d shift %d: %s\n", mode, shift, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 64; ++n) {
          float ref = 0;
          for (int k = 0; k < K; ++k) ref += fa[(m + shift) * K + k] * fb[n * K + k];
          if (fabsf(ref - got[m * 64 + n]) > 1e-3f) ++bad;
        }
      printf("base_offset %s shift %2d: %d / %d wrong\n", mode ? "set " : "zero", shift, bad, 128 * 64);
    }
  return 0;
}
