// Host side of the GPU expf / SiLU sweep (tests/test_gpu_expf.py): counts the
// float results that differ in bits from the live host libm (expf, or the
// reference's SiLU x / (1 + expf(-x)), proj/src/eltwise.cpp:31-34) over the
// bit patterns first .. first+n-1. NaN == NaN. Built -ffp-contract=off like
// the reference (CMakeLists.txt:13).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

extern "C" unsigned long long expf_check(const float* got, uint32_t first, unsigned long long n, int mode,
                                         unsigned long long* first_bad) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  std::vector<unsigned long long> bad(nt, 0), where(nt, ~0ull);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const unsigned long long lo = n * t / nt, hi = n * (t + 1) / nt;
      for (unsigned long long i = lo; i < hi; ++i) {
        const uint32_t u = first + static_cast<uint32_t>(i);
        float x;
        std::memcpy(&x, &u, 4);
        volatile float e = mode == 0 ? expf(x) : expf(-x);
        const float want = mode == 0 ? e : x / (1.0f + e);
        uint32_t a, b;
        std::memcpy(&a, &want, 4);
        std::memcpy(&b, &got[i], 4);
        if (a != b && !(std::isnan(want) && std::isnan(got[i]))) {
          if (where[t] == ~0ull) where[t] = i;
          ++bad[t];
        }
      }
    });
  for (auto& x : th) x.join();
  unsigned long long tot = 0;
  *first_bad = ~0ull;
  for (unsigned t = 0; t < nt; ++t) {
    tot += bad[t];
    if (where[t] < *first_bad) *first_bad = where[t];
  }
  return tot;
}
