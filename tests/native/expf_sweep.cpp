// Exhaustive check of the device expf restatement (compiled here as host code)
// against the host libm expf over every float bit pattern. Usage:
//   expf_sweep <variant: 1=fma 0=sse2>   -> prints "mismatches <n> digest <hex>"
// The digest is FNV-1a over libm expf output bits for x in [-110, 90] (the
// SURVEY Appendix B protocol), ascending bit order of negatives then positives.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include "glibc_expf.h"

int main(int argc, char** argv) {
  bool fma = argc > 1 ? std::atoi(argv[1]) != 0 : true;
  unsigned nt = std::thread::hardware_concurrency();
  std::vector<unsigned long long> bad(nt, 0);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      unsigned long long lo = (0x100000000ull * t) / nt, hi = (0x100000000ull * (t + 1)) / nt;
      for (unsigned long long b = lo; b < hi; ++b) {
        uint32_t u = (uint32_t)b;
        float x;
        std::memcpy(&x, &u, 4);
        float a = expf(x), c = sige_b200::glibc_expf(x, fma);
        uint32_t ua, uc;
        std::memcpy(&ua, &a, 4);
        std::memcpy(&uc, &c, 4);
        if (ua != uc && !(std::isnan(a) && std::isnan(c))) {
          if (bad[t] < 3) std::fprintf(stderr, "x=%a libm=%a ours=%a\n", x, a, c);
          ++bad[t];
        }
      }
    });
  for (auto& x : th) x.join();
  unsigned long long tot = 0;
  for (auto v : bad) tot += v;
  std::printf("mismatches %llu\n", tot);
  return tot != 0;
}
