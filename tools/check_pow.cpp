// CPU check of the restated pow(h, 4/3) (paper_1807_00672_b200/csrc/swe_pow.cuh)
// against the host libm pow, over N samples.  Usage: check_pow [N] [seed]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include "swe_pow.cuh"
int main(int argc, char** argv) {
  const long n = argc > 1 ? atol(argv[1]) : 10000000;
  std::mt19937_64 rng(argc > 2 ? atol(argv[2]) : 1);
  std::uniform_real_distribution<double> le(std::log(1e-300), std::log(1e300));
  std::uniform_real_distribution<double> lp(std::log(1e-7), std::log(1e4));
  long bad = 0;
  auto check = [&](double x) {
    const double a = swe_b200::swe_pow43(x), b = std::pow(x, 4.0 / 3.0);
    uint64_t ua, ub;
    std::memcpy(&ua, &a, 8);
    std::memcpy(&ub, &b, 8);
    if (ua != ub && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 10) std::printf("MISMATCH x=%a mine=%a libm=%a\n", x, a, b);
      ++bad;
    }
  };
  for (double x : {0.0, -0.0, 1.0, 2.0, 1e-6, 1e-300, 5e-324, 1e-310, (double)INFINITY, (double)NAN, -1.0, 8.0, 27.0, 1e100, 1e200, 1e-200})
    check(x);
  for (long i = 0; i < n; ++i) check(std::exp(i & 1 ? lp(rng) : le(rng)));
  // every ulp around 1 and a dense sweep of [h_dry, 10]
  double x = 1.0;
  for (int i = 0; i < 100000; ++i) { check(x); x = std::nextafter(x, 2.0); }
  x = 1.0;
  for (int i = 0; i < 100000; ++i) { check(x); x = std::nextafter(x, 0.0); }
  std::printf("checked %ld samples: %ld mismatches\n", n + 200016, bad);
  return bad != 0;
}
