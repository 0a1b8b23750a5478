// common.cpp — errors, launch accounting, device queries, epilogue conversion.
#include "common.hpp"

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

namespace sige_b200 {

std::atomic<uint64_t> g_launches{0};

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                  ") at " + file + ":" + std::to_string(line) + ": " + what);
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess)
      return v;
    return 148;
  }();
  return n;
}

// Which glibc expf build this host's libm dispatches to: the two builds
// differ on a handful of inputs (found by the exhaustive sweep in
// tests/native/expf_sweep.cpp); x = 0x1.04845ep+5 is one of them.
bool host_expf_is_fma() {
  static bool fma = [] {
    volatile float x = 0x1.04845ep+5f;
    float libm = expf(x);
    float via_fma = glibc_expf(x, true), via_sse2 = glibc_expf(x, false);
    uint32_t a, b, c;
    std::memcpy(&a, &libm, 4);
    std::memcpy(&b, &via_fma, 4);
    std::memcpy(&c, &via_sse2, 4);
    if (a == c && a != b) return false;
    return true;  // FMA build (or a libm matching neither: documented in DESIGN.md)
  }();
  return fma;
}

DevEpilogue make_dev_epilogue(const sige_epilogue* e, int channels, int batch) {
  DevEpilogue d;
  d.fma_expf = host_expf_is_fma() ? 1 : 0;
  if (!e) return d;
  if (e->num_steps < 0 || e->num_steps > SIGE_MAX_EPI_STEPS)
    throw ConfigError("epilogue: at most " + std::to_string(SIGE_MAX_EPI_STEPS) + " steps");
  for (int i = 0; i < e->num_steps; ++i) {
    const sige_epilogue_step& s = e->steps[i];
    d.kind[i] = s.kind;
    if (s.kind == SIGE_EPI_ACTIVATION) {
      if (s.act < SIGE_ACT_NONE || s.act > SIGE_ACT_SILU)
        throw ConfigError("unknown activation: " + std::to_string(s.act));
      d.act[i] = s.act;
    } else if (s.kind == SIGE_EPI_SCALE_SHIFT) {
      // param_slice (eltwise.cpp:48-58): C values broadcast, N*C per sample.
      if (s.nparams == channels) {
        d.per_sample[i] = 0;
      } else if (channels > 0 && s.nparams % channels == 0 && batch * channels <= s.nparams) {
        d.per_sample[i] = 1;
      } else {
        throw ConfigError("epilogue: affine param size " + std::to_string(s.nparams) +
                          " does not match channels " + std::to_string(channels));
      }
      if (!s.scale || !s.shift) throw ConfigError("epilogue: null scale/shift");
      d.scale[i] = s.scale;
      d.shift[i] = s.shift;
    } else {
      throw ConfigError("epilogue: unknown step kind " + std::to_string(s.kind));
    }
  }
  d.num_steps = e->num_steps;
  return d;
}

}  // namespace sige_b200
