// swe_pow.cuh -- h^(4/3) for the Manning friction denominator, bit-identical
// to the reference's std::pow(u.h, 4.0 / 3.0) (kernels.hpp:197).
//
// std::pow resolves to the host glibc (2.39-0ubuntu8.5 in this image), whose
// ifunc picks __pow_fma on every FMA+AVX2 x86-64 host.  That routine is
// glibc's sysdeps/ieee754/dbl-64/e_pow.c (ARM optimized-routines): a
// table-driven log with ~15 extra bits (log_inline) and a table-driven exp
// (exp_inline), compiled with __FP_FAST_FMA and GCC's default FP contraction.
// The operation sequence below restates the fast path of that binary
// instruction for instruction (libm+0x7a1e0: every vfmadd/vfmsub is an fma()
// here, every vaddsd/vsubsd/vmulsd a plain op; this TU is built with
// --fmad=false so nvcc adds no contraction of its own), with the two data
// tables copied from the installed libm by tools/gen_pow_tables.py.  Inputs
// off the fast path: zero/inf/nan and negative x follow glibc's rules;
// subnormal x is normalised as glibc does; results that would under/overflow
// (|4/3 ln h| >= 512, i.e. h outside (1e-166, 1e166)) use CUDA's pow.
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

#include "swe_pow_tables.h"

#if defined(__CUDACC__)
#define SWE_HD __host__ __device__ __forceinline__
#else
#define SWE_HD inline
#endif

namespace swe_b200 {

#if defined(__CUDACC__)
__device__ const unsigned long long g_pow_log_tab[128][3] = SWE_POW_LOG_TAB;
__device__ const unsigned long long g_pow_exp_tab[256] = SWE_POW_EXP_TAB;
#endif
static const unsigned long long h_pow_log_tab[128][3] = SWE_POW_LOG_TAB;
static const unsigned long long h_pow_exp_tab[256] = SWE_POW_EXP_TAB;

SWE_HD double pw_as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  std::memcpy(&d, &u, 8);
  return d;
#endif
}

SWE_HD uint64_t pw_as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
#endif
}

SWE_HD uint64_t pw_log_tab(int i, int k) {
#if defined(__CUDA_ARCH__)
  return __ldg(&g_pow_log_tab[i][k]);
#else
  return h_pow_log_tab[i][k];
#endif
}

SWE_HD uint64_t pw_exp_tab(int i) {
#if defined(__CUDA_ARCH__)
  return __ldg(&g_pow_exp_tab[i]);
#else
  return h_pow_exp_tab[i];
#endif
}

SWE_HD double pw_fma(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

// log(x) = hi + lo for the bit pattern ix of a positive normal x
// (e_pow.c log_inline; libm+0x7a228..0x7a329).
SWE_HD void pw_log_inline(uint64_t ix, double* hi_out, double* lo_out) {
  const double Ln2hi = 0x1.62e42fefa3800p-1, Ln2lo = 0x1.ef35793c76730p-45;
  const double A0 = -0x1p-1, A1 = -0x1.5555555555560p-1, A2 = 0x1.0000000000006p-1,
               A3 = 0x1.999999959554ep-1, A4 = -0x1.555555529a47ap-1,
               A5 = -0x1.2495b9b4845e9p+0, A6 = 0x1.0002b8b263fc3p+0;
  const uint64_t tmp = ix - 0x3fe6955500000000ull;  // ix - OFF
  const int i = (int)((tmp >> 45) & 127);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double z = pw_as_double(iz);
  const double kd = (double)k;
  const double invc = pw_as_double(pw_log_tab(i, 0));
  const double logc = pw_as_double(pw_log_tab(i, 1));
  const double logctail = pw_as_double(pw_log_tab(i, 2));

  const double t1 = pw_fma(kd, Ln2hi, logc);
  const double lo1 = pw_fma(kd, Ln2lo, logctail);
  const double r = pw_fma(z, invc, -1.0);
  const double ar = r * A0;
  const double p1 = pw_fma(r, A2, A1);
  const double p3 = pw_fma(r, A4, A3);
  const double t2 = r + t1;
  const double lo2 = (t1 - t2) + r;
  const double ar2 = r * ar;
  const double ar3 = r * ar2;
  const double lo3 = pw_fma(ar, r, -ar2);
  const double hi = t2 + ar2;
  const double p5 = pw_fma(r, A6, A5);
  const double q = pw_fma(p5, ar2, p3);
  const double lo4 = (t2 - hi) + ar2;
  const double poly = pw_fma(ar2, q, p1);
  double s = lo1 + lo2;
  s = s + lo3;
  s = s + lo4;
  const double lo = pw_fma(ar3, poly, s);
  const double y = hi + lo;
  *lo_out = (hi - y) + lo;
  *hi_out = y;
}

SWE_HD double swe_pow43(double x) {
  const double Y = 4.0 / 3.0;
  uint64_t ix = pw_as_u64(x);
  const uint32_t topx = (uint32_t)(ix >> 52);
  if (topx - 1u >= 0x7feu) {  // zero / subnormal / inf / nan / negative
    if (2 * ix - 1 >= 2 * 0x7ff0000000000000ull - 1) return x * x;  // 0, inf, nan
    if (ix >> 63) return (x - x) / (x - x);  // finite x < 0, non-integer y: NaN
    // positive subnormal: normalise so the exponent goes negative
    ix = pw_as_u64(x * 0x1p52) & 0x7fffffffffffffffull;
    ix -= 52ull << 52;
  }
  double lhi, llo;
  pw_log_inline(ix, &lhi, &llo);
  const double ehi = Y * lhi;
  const double elo = pw_fma(Y, llo, pw_fma(lhi, Y, -ehi));

  // exp_inline(ehi, elo, 0) (libm+0x7a332..0x7a404)
  const uint32_t abstop = (uint32_t)(pw_as_u64(ehi) >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {
    if (abstop - 0x3c9u >= 0x80000000u) return 1.0 + ehi;  // |ehi| < 2^-54
    if (abstop >= 0x409u) return (pw_as_u64(ehi) >> 63) ? 0.0 : INFINITY;
#if defined(__CUDA_ARCH__)
    return pow(x, Y);  // scale near the range ends (glibc specialcase)
#else
    return std::pow(x, Y);
#endif
  }
  const double InvLn2N = 0x1.71547652b82fep7, Shift = 0x1.8p52;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3, C4 = 0x1.55555cf172b91p-5,
               C5 = 0x1.1111167a4d017p-7;
  double kd = pw_fma(ehi, InvLn2N, Shift);
  const uint64_t ki = pw_as_u64(kd);
  kd = kd - Shift;
  double r = pw_fma(kd, NegLn2loN, pw_fma(kd, NegLn2hiN, ehi));
  r = elo + r;
  const int idx = 2 * (int)(ki & 127);
  const uint64_t top = ki << 45;
  const double tail = pw_as_double(pw_exp_tab(idx));
  const uint64_t sbits = pw_exp_tab(idx + 1) + top;
  const double r2 = r * r;
  const double a = pw_fma(r2, pw_fma(r, C3, C2), tail + r);
  const double tmp = pw_fma(r2 * r2, pw_fma(r, C5, C4), a);
  const double scale = pw_as_double(sbits);
  return pw_fma(tmp, scale, scale);
}

}  // namespace swe_b200
