// glibc_expf.h — bit-exact restatement of glibc 2.28+ `expf` for device code.
//
// The reference's SiLU is `x / (1 + std::exp(-x))` (proj/src/eltwise.cpp:31-34),
// i.e. glibc libm `expf`. glibc selects one of two builds of the same source
// (sysdeps/ieee754/flt-32/e_expf.c) at load time by ifunc: an SSE2 build
// (separately rounded multiply/add) and an FMA build compiled with -mfma, where
// GCC contracted `z = InvLn2N*x` into both of its uses and fused the three
// polynomial steps. Read off the host libm.so.6 (glibc 2.39) disassembly:
//
//   SSE2: z=I*x; k=S+z; kd=k-S; r=z-kd; p0=C0*r+C1; p2=C2*r+1; y=p0*(r*r)+p2
//   FMA : k=fma(I,x,S); kd=k-S; r=fma(I,x,-kd); p0=fma(r,C0,C1);
//         p2=fma(r,C2,1); y=fma(p0,r*r,p2)
//   both: s = asdouble(T[k&31] + (k<<47)); return (float)(y*s)
//
// with |x| >= 88 handled by the special cases below. Both variants are checked
// against the live host libm over all 2^32 inputs by the test suite
// (tests/test_expf.py and the GPU sweep in tests/test_gpu_ops.py).
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define SIGE_HD __host__ __device__ __forceinline__
#else
#define SIGE_HD inline
#endif

namespace sige_b200 {

// __exp2f_data.tab (32 entries): asuint64(2^(i/32)) - (i << 52)/32.
#define SIGE_EXP2F_TAB { \
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull, \
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, \
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull, \
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull, \
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull, \
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull, \
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull, \
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull, \
}
static const uint64_t kExp2fTabHost[32] = SIGE_EXP2F_TAB;
#ifdef __CUDACC__
// Global (not __constant__): the index k & 31 differs per lane, and the
// constant cache serialises divergent indices (up to 32 ways per warp load);
// through L1 the whole 256-byte table is two cache lines.
__device__ const uint64_t kExp2fTabDev[32] = SIGE_EXP2F_TAB;
#endif


namespace expf_detail {
constexpr double kInvLn2N = 0x1.71547652b82fep+5;  // invln2_scaled = 1/ln2 * 32
constexpr double kShift = 0x1.8p+52;
constexpr double kC0 = 0x1.c6af84b912394p-20;  // poly_scaled
constexpr double kC1 = 0x1.ebfce50fac4f3p-13;
constexpr double kC2 = 0x1.62e42ff0c52d6p-6;

SIGE_HD uint32_t f2u(float x) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(x);
#else
  union {
    float f;
    uint32_t u;
  } v;
  v.f = x;
  return v.u;
#endif
}
SIGE_HD float u2f(uint32_t x) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(x);
#else
  union {
    float f;
    uint32_t u;
  } v;
  v.u = x;
  return v.f;
#endif
}
SIGE_HD uint64_t d2u(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  union {
    double d;
    uint64_t u;
  } v;
  v.d = x;
  return v.u;
#endif
}
SIGE_HD double u2d(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(x));
#else
  union {
    double d;
    uint64_t u;
  } v;
  v.u = x;
  return v.d;
#endif
}
// Separately rounded double ops (no contraction regardless of compiler flags).
SIGE_HD double dmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  volatile double r = a * b;
  return r;
#endif
}
SIGE_HD double dadd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  volatile double r = a + b;
  return r;
#endif
}
SIGE_HD double dfma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return __builtin_fma(a, b, c);
#endif
}
SIGE_HD uint64_t tab(uint32_t i) {
#ifdef __CUDA_ARCH__
  return __ldg(kExp2fTabDev + i);
#else
  return kExp2fTabHost[i];
#endif
}
}  // namespace expf_detail

// fma_variant: true reproduces __expf_fma (the ifunc choice on any host with
// FMA+AVX2), false reproduces the SSE2 build.
SIGE_HD float glibc_expf(float x, bool fma_variant) {
  using namespace expf_detail;
  const uint32_t ix = f2u(x);
  const uint32_t abstop = (ix >> 20) & 0x7ffu;
  if (abstop >= 0x42bu) {  // |x| >= 88 or not finite
    if (ix == 0xff800000u) return 0.0f;
    if (abstop >= 0x7f8u) return x + x;
    if (x > 0x1.62e42ep6f) return u2f(0x7f800000u);  // __math_oflowf: 0x1p97f^2 = +inf
    if (x < -0x1.9fe368p6f) return 0.0f;                 // __math_uflowf: 0x1p-95f^2
    if (x < -0x1.9d1d9ep6f) return 0x1p-149f;            // __math_may_uflowf: 0x1.4p-75f^2
  }
  const double xd = static_cast<double>(x);
  double k, kd, r, y;
  if (fma_variant) {
    k = dfma(kInvLn2N, xd, kShift);
    kd = dadd(k, -kShift);
    r = dfma(kInvLn2N, xd, -kd);
  } else {
    const double z = dmul(kInvLn2N, xd);
    k = dadd(kShift, z);
    kd = dadd(k, -kShift);
    r = dadd(z, -kd);
  }
  const uint64_t ki = d2u(k);
  const double s = u2d(tab(static_cast<uint32_t>(ki & 31u)) + (ki << 47));
  const double r2 = dmul(r, r);
  if (fma_variant) {
    const double p0 = dfma(r, kC0, kC1);
    const double p2 = dfma(r, kC2, 1.0);
    y = dfma(p0, r2, p2);
  } else {
    const double p0 = dadd(dmul(kC0, r), kC1);
    const double p2 = dadd(dmul(kC2, r), 1.0);
    y = dadd(dmul(p0, r2), p2);
  }
  y = dmul(y, s);
#ifdef __CUDA_ARCH__
  return __double2float_rn(y);
#else
  return static_cast<float>(y);
#endif
}

}  // namespace sige_b200
