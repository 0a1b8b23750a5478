// common.hpp — shared host/device infrastructure of libsige_b200.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "glibc_expf.h"
#include "sige_b200.h"

namespace sige_b200 {

// ConfigError of the reference (proj/include/sige/common.hpp:14-17): every
// geometry / configuration violation. Mapped to SIGE_ERR_CONFIG at the C ABI.
class ConfigError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define SIGE_CUDA(x)                                                      \
  do {                                                                    \
    cudaError_t e_ = (x);                                                 \
    if (e_ != cudaSuccess) ::sige_b200::throw_cuda(e_, #x, __FILE__, __LINE__); \
  } while (0)

// Every kernel launch goes through this so the library can report how many of
// its own kernels ran (sige_kernel_launch_count) and fail loudly on launch errors.
extern std::atomic<uint64_t> g_launches;
inline void after_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw_cuda(e, name, __FILE__, __LINE__);
}

// True the first time it is called for the current device (per flag word):
// function attributes such as the dynamic shared-memory limit are per device
// context, so an engine on a second GPU must set them again.
inline bool first_on_device(std::atomic<uint64_t>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const uint64_t bit = 1ull << dev;
  return (done.fetch_or(bit) & bit) == 0;
}

inline cudaStream_t as_stream(sige_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

inline int conv_out_dim(int in, int k, int stride) {
  int pad = (k - 1) / 2;
  return (in + 2 * pad - k) / stride + 1;
}

// Which glibc expf build the host uses (decides SiLU bits). Probed once from
// the live libm by the C ABI layer (see capi.cpp: detect_expf_variant).
bool host_expf_is_fma();

// Number of SMs of the current device (cached).
int sm_count();

// ---------------------------------------------------------------- epilogue
// Device form of `sige::Epilogue` (proj/include/sige/eltwise.hpp:30-59): up
// to SIGE_MAX_EPI_STEPS ordered steps, each a per-channel ScaleShift (with C
// or N*C params, eltwise.cpp:48-58) or an activation. Passed by value.
struct DevEpilogue {
  int num_steps = 0;
  int fma_expf = 1;  // glibc expf variant to reproduce
  // 1: SiLU as x / (1 + __expf(-x)) with the fast divide (tensor-core modes,
  // whose operands are rounded to 10-bit mantissas anyway); 0: bit-exact
  // glibc expf + IEEE divide (the reference's arithmetic, exact mode).
  int fast = 0;
  int kind[SIGE_MAX_EPI_STEPS] = {};
  int act[SIGE_MAX_EPI_STEPS] = {};
  int per_sample[SIGE_MAX_EPI_STEPS] = {};  // 1 if params are N*C (sample-major)
  const float* scale[SIGE_MAX_EPI_STEPS] = {};
  const float* shift[SIGE_MAX_EPI_STEPS] = {};
};

// Validates and converts a C-ABI epilogue for `channels` and `batch`, with
// the reference's "epilogue: affine param size ..." message (eltwise.cpp:55-57).
DevEpilogue make_dev_epilogue(const sige_epilogue* e, int channels, int batch);

#ifdef __CUDACC__
// Reference activation arithmetic (eltwise.cpp:23-36), no FMA contraction.
__device__ __forceinline__ float dev_act(float v, int kind, int fma_expf, int fast = 0) {
  if (kind == SIGE_ACT_RELU) return v > 0.0f ? v : 0.0f;  // NaN -> 0, -0 -> +0
  if (kind == SIGE_ACT_LEAKY_RELU) return v > 0.0f ? v : __fmul_rn(0.2f, v);  // SPADE blocks (config 3)
  if (kind == SIGE_ACT_SILU && fast) return __fdividef(v, 1.0f + __expf(-v));
  if (kind == SIGE_ACT_SILU) {
    float e = glibc_expf(-v, fma_expf != 0);
    return __fdiv_rn(v, __fadd_rn(1.0f, e));
  }
  return v;
}

// Applies the chain to one value of channel ch of sample n (apply_span /
// apply_cell / apply_slab are all per-value maps, eltwise.cpp:110-150).
__device__ __forceinline__ float dev_epi(const DevEpilogue& e, float v, int ch, int channels,
                                         int n) {
#pragma unroll
  for (int s = 0; s < SIGE_MAX_EPI_STEPS; ++s) {
    if (s >= e.num_steps) break;
    if (e.kind[s] == SIGE_EPI_ACTIVATION) {
      v = dev_act(v, e.act[s], e.fma_expf, e.fast);
    } else {
      int off = e.per_sample[s] ? n * channels + ch : ch;
      v = __fadd_rn(__fmul_rn(__ldg(e.scale[s] + off), v), __ldg(e.shift[s] + off));
    }
  }
  return v;
}

// The chain over CNT consecutive channels ch0.. of one pixel, same arithmetic
// as dev_epi per value; the per-channel params of each step are fetched with
// 16-byte loads up front (one memory round trip per step instead of one per
// value) when the offsets are 4-aligned.
template <int CNT>
__device__ __forceinline__ void dev_epi_vec(const DevEpilogue& e, float* v, int ch0, int channels, int n) {
  static_assert(CNT % 4 == 0, "CNT must be a multiple of 4");
#pragma unroll
  for (int s = 0; s < SIGE_MAX_EPI_STEPS; ++s) {
    if (s >= e.num_steps) break;
    if (e.kind[s] == SIGE_EPI_ACTIVATION) {
#pragma unroll
      for (int j = 0; j < CNT; ++j) v[j] = dev_act(v[j], e.act[s], e.fma_expf, e.fast);
    } else {
      const int off = e.per_sample[s] ? n * channels + ch0 : ch0;
      float sc[CNT], sh[CNT];
      if ((off & 3) == 0) {
#pragma unroll
        for (int j = 0; j < CNT; j += 4) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(e.scale[s] + off + j));
          const float4 b = __ldg(reinterpret_cast<const float4*>(e.shift[s] + off + j));
          sc[j] = a.x, sc[j + 1] = a.y, sc[j + 2] = a.z, sc[j + 3] = a.w;
          sh[j] = b.x, sh[j + 1] = b.y, sh[j + 2] = b.z, sh[j + 3] = b.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < CNT; ++j) {
          sc[j] = __ldg(e.scale[s] + off + j);
          sh[j] = __ldg(e.shift[s] + off + j);
        }
      }
#pragma unroll
      for (int j = 0; j < CNT; ++j) v[j] = __fadd_rn(__fmul_rn(sc[j], v[j]), sh[j]);
    }
  }
}
#endif

}  // namespace sige_b200
