// swe_phys.cuh -- FP64 point physics of the explicit HLLC step, device side.
//
// Same operations in the same operand order as the reference's host physics
// (/root/reference/proj/include/swe/kernels.hpp, cited per function); where
// the reference branches, the alternatives are evaluated and the branch's
// value selected (SIMT), so the device result is bit-identical: the translation
// unit is compiled with --fmad=false (the reference builds with
// -ffp-contract=off, CMakeLists.txt:17-18), every + - * / sqrt is an IEEE
// round-to-nearest FP64 op on both sides, and std::min / std::max are spelled
// out as the (b<a)?b:a / (a<b)?b:a selections they are (signed zeros, NaN).
// The one libm call, pow(h, 4/3), goes through swe_pow43 (swe_pow.cuh).
#pragma once

#include "swe_pow.cuh"

namespace swe_b200 {

struct Phys {
  double g, h_dry, cfl, dt_max, h_ref;
};

struct Cons {
  double h, qx, qy;
};

struct Flux {
  double m, fx, fy;  // mass, x-momentum, y-momentum per unit length
};

__device__ __forceinline__ double sel_min(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double sel_max(double a, double b) { return (a < b) ? b : a; }

// IEEE a / b and sqrt(x) that keep zero operands off CUDA's out-of-line
// special-operand paths.  The inline fast path of div.rn.f64 rejects
// numerators below 2^-969 -- zero included -- so every still-water momentum
// (q = 0) and symmetric contact (num = 0) called the slow subroutine; ncu
// (profiles/r01_*): 33% of k_tile's executed instructions, 3.06M calls per
// 10M-cell step.  The operand is swapped for 1.0 before an opaque div.rn /
// sqrt.rn (plain C++ lets nvcc fold the select away) and the exact IEEE
// answer selected afterwards: for a == +-0 and finite non-zero b, a / b is
// the signed zero a * b; sqrt(+-0) = +-0.
#ifndef SWE_ZERO_SAFE
#define SWE_ZERO_SAFE 1
#endif
// velocity quotients as warp-uniform branches (dry or still cells skip the
// division) rather than selects: measured -0.1..-2.8% and fewer spills
#ifndef SWE_VEL_BRANCH
#define SWE_VEL_BRANCH 1
#endif
__device__ __forceinline__ double div_rn(double a, double b) {
  double q;
  asm("div.rn.f64 %0, %1, %2;" : "=d"(q) : "d"(a), "d"(b));
  return q;
}
__device__ __forceinline__ double qdiv(double a, double b) {
#if SWE_ZERO_SAFE
  const bool z = (a == 0.0) && isfinite(b) && (b != 0.0);
  const double q = div_rn(z ? 1.0 : a, b);
  return z ? a * b : q;
#else
  return a / b;
#endif
}
// a / b for b known positive and finite (depths >= h_dry > 0, friction
// denominators >= 1): only the numerator needs the guard (0 / b = a)
__device__ __forceinline__ double qdivp(double a, double b) {
#if SWE_VEL_BRANCH
  if (a == 0.0) return a;  // warps at rest skip the division
  return div_rn(a, b);
#elif SWE_ZERO_SAFE
  const bool z = a == 0.0;
  const double q = div_rn(z ? 1.0 : a, b);
  return z ? a : q;
#else
  return a / b;
#endif
}
__device__ __forceinline__ double qsqrt(double x) {
#if SWE_ZERO_SAFE
  const bool z = x == 0.0;
  double r;
  asm("sqrt.rn.f64 %0, %1;" : "=d"(r) : "d"(z ? 1.0 : x));
  return z ? x : r;
#else
  return sqrt(x);
#endif
}

// velocity(), kernels.hpp:15-18: dry cells move with zero velocity.  The
// quotient is formed against a safe denominator so a dry (h = 0) lane never
// takes the division's special-operand slow path; the selected value is the
// reference's exactly.
__device__ __forceinline__ void vel(const Cons& u, double h_dry, double& vx, double& vy) {
#if SWE_VEL_BRANCH
  // a branch, not a select: warps of dry cells skip the divisions
  vx = 0.0;
  vy = 0.0;
  if (!(u.h < h_dry)) {
    vx = qdivp(u.qx, u.h);
    vy = qdivp(u.qy, u.h);
  }
#else
  const bool dry = u.h < h_dry;
  const double hs = dry ? 1.0 : u.h;
  vx = dry ? 0.0 : qdivp(u.qx, hs);
  vy = dry ? 0.0 : qdivp(u.qy, hs);
#endif
}

// physical_flux_normal(), kernels.hpp:21-27.
__device__ __forceinline__ Flux normal_flux(const Cons& u, double nx, double ny, const Phys& P) {
  if (u.h < P.h_dry) return Flux{0.0, 0.0, 0.0};
  const double vx = qdivp(u.qx, u.h), vy = qdivp(u.qy, u.h);
  const double un = vx * nx + vy * ny;
  const double p = ((0.5 * P.g) * u.h) * u.h;
  return Flux{u.h * un, ((u.h * vx) * un) + p * nx, ((u.h * vy) * un) + p * ny};
}

// hllc_flux(), kernels.hpp:72-114, with wave_speed_estimates() (:38-66)
// inlined and restructured for SIMT: the dry-front / two-rarefaction speed
// branches and the three flux branches are all evaluated and selected, so a
// warp never serialises them.  Each selected value is produced by exactly the
// expression the reference's branch uses, hence bit-identical results; the
// both-dry and identical-state early outs stay branches (spatially coherent).
__device__ __forceinline__ Flux hllc(const Cons& L, const Cons& R, double nx, double ny,
                                         const Phys& P) {
  const bool dryL = L.h < P.h_dry, dryR = R.h < P.h_dry;
  if (dryL && dryR) return Flux{0.0, 0.0, 0.0};
  if (L.h == R.h && L.qx == R.qx && L.qy == R.qy) return normal_flux(L, nx, ny, P);

  double vLx, vLy, vRx, vRy;
  vel(L, P.h_dry, vLx, vLy);
  vel(R, P.h_dry, vRx, vRy);
  const double unL = vLx * nx + vLy * ny, utL = (-vLx) * ny + vLy * nx;
  const double unR = vRx * nx + vRy * ny, utR = (-vRx) * ny + vRy * nx;
  const double hL = L.h, hR = R.h;

  // kernels.hpp:45-59; a dry side's root is taken of a dummy positive value
  const double cL = sqrt(P.g * (dryL ? 1.0 : hL));
  const double cR = sqrt(P.g * (dryR ? 1.0 : hR));
  const double us = ((0.5 * (unL + unR)) + cL) - cR;
  const double cs = fabs((0.5 * (cL + cR)) + (0.25 * (unL - unR)));
  double SL = sel_min(unL - cL, us - cs);
  double SR = sel_max(unR + cR, us + cs);
  const bool frontR = dryR && !dryL, frontL = dryL && !dryR;
  SL = frontR ? unL - cL : (frontL ? unR - 2.0 * cR : SL);
  SR = frontR ? unL + 2.0 * cL : (frontL ? unR + cR : SR);

  const double aR = unR - SR, aL = unL - SL;
  const double num = ((SL * hR) * aR) - ((SR * hL) * aL);
  const double den = (hR * aR) - (hL * aL);
  const bool tiny = fabs(den) < 1e-14;
  const double Ss = tiny ? 0.5 * (unL + unR) : qdiv(num, tiny ? 1.0 : den);

  const double FL0 = hL * unL, FL1 = ((hL * unL) * unL) + (((0.5 * P.g) * hL) * hL);
  const double FR0 = hR * unR, FR1 = ((hR * unR) * unR) + (((0.5 * P.g) * hR) * hR);
  // SL < SR always (both-dry excluded), so the fan quotient is always safe
  const double inv = 1.0 / (SR - SL);
  const double sls = SL * SR;
  const double f0s = (((SR * FL0) - (SL * FR0)) + (sls * (hR - hL))) * inv;
  const double f1s = (((SR * FL1) - (SL * FR1)) + (sls * ((hR * unR) - (hL * unL)))) * inv;
  const bool left = SL >= 0.0, right = !left && SR <= 0.0;
  const double f0 = left ? FL0 : (right ? FR0 : f0s);
  const double f1 = left ? FL1 : (right ? FR1 : f1s);
  const double ft = f0 * (left ? utL : (right ? utR : (Ss >= 0.0 ? utL : utR)));
  return Flux{f0, (f1 * nx) - (ft * ny), (f1 * ny) + (ft * nx)};
}

// wall_flux(), kernels.hpp:156-164: Riemann problem against the mirror state,
// mass pinned to zero.
__device__ __forceinline__ Flux wall(const Cons& u, double nx, double ny, const Phys& P) {
  double vx, vy;
  vel(u, P.h_dry, vx, vy);
  const double un = vx * nx + vy * ny;
  const Cons m{u.h, u.h * (vx - ((2.0 * un) * nx)), u.h * (vy - ((2.0 * un) * ny))};
  Flux f = hllc(u, m, nx, ny, P);
  f.m = 0.0;
  return f;
}

// One interior edge of compute_fluxes() (engine.hpp:161-166) with
// hydrostatic_reconstruct() (kernels.hpp:126-152): the applied left flux
// {f0, fmx + pl nx, fmy + pl ny} and the right flux's momentum part
// {-(fmx + pr nx), -(fmy + pr ny)}; the right mass is -f0.  For SIMT: only
// the lower side can be cut (hls != h needs
// zl < zr, hrs != h needs zr < zl), so the one candidate side's velocity is
// computed unconditionally on a selected state instead of in two divergent
// branches (finite bathymetry is a swe_dev_create precondition).
__device__ __forceinline__ void interior_edge(const Cons& uL, double zl, const Cons& uR,
                                                  double zr, double nx, double ny, const Phys& P,
                                                  double& f0, double& lx, double& ly, double& rx,
                                                  double& ry) {
  const double hls = zl >= zr ? uL.h : sel_max(0.0, uL.h + (zl - zr));
  const double hrs = zr >= zl ? uR.h : sel_max(0.0, uR.h + (zr - zl));
  const bool sideL = zl < zr;
  const Cons us = sideL ? uL : uR;
  const double hcut = sideL ? hls : hrs;
  double vx, vy;
  vel(us, P.h_dry, vx, vy);
  const Cons cut{hcut, hcut * vx, hcut * vy};
  const Cons a = (hls == uL.h) ? uL : cut;
  const Cons b = (hrs == uR.h) ? uR : cut;
  const double pl = (0.5 * P.g) * ((uL.h * uL.h) - (hls * hls));
  const double pr = (0.5 * P.g) * ((uR.h * uR.h) - (hrs * hrs));
  const Flux f = hllc(a, b, nx, ny, P);
  f0 = f.m;
  lx = f.fx + pl * nx;
  ly = f.fy + pl * ny;
  rx = -(f.fx + pr * nx);
  ry = -(f.fy + pr * ny);
}

// apply_friction(), kernels.hpp:191-199 (semi-implicit Manning).
__device__ __forceinline__ Cons friction(const Cons& u, double n, double dt, const Phys& P) {
  if (u.h < P.h_dry || n == 0.0) return u;
  const double vx = qdivp(u.qx, u.h), vy = qdivp(u.qy, u.h);
  const double s = qsqrt(vx * vx + vy * vy);
  if (s == 0.0) return u;
  const double den = 1.0 + (((((dt * P.g) * n) * n) * s) / swe_pow43(u.h));
  return Cons{u.h, qdivp(u.qx, den), qdivp(u.qy, den)};
}

// wave_speed_estimates(), kernels.hpp:38-66, as its own entry point (the
// point API; hllc() above carries a select-form copy for the step kernels)
__device__ __forceinline__ void wave_speeds(double hL, double uL, double hR, double uR,
                                            const Phys& P, double& SL, double& Ss, double& SR) {
  const double g = P.g;
  const bool dryL = hL < P.h_dry, dryR = hR < P.h_dry;
  if (dryR && !dryL) {
    const double cL = sqrt(g * hL);
    SL = uL - cL;
    SR = uL + 2.0 * cL;
  } else if (dryL && !dryR) {
    const double cR = sqrt(g * hR);
    SL = uR - 2.0 * cR;
    SR = uR + cR;
  } else {
    const double cL = sqrt(g * hL);
    const double cR = sqrt(g * hR);
    const double us = ((0.5 * (uL + uR)) + cL) - cR;
    const double cs = fabs((0.5 * (cL + cR)) + (0.25 * (uL - uR)));
    SL = sel_min(uL - cL, us - cs);
    SR = sel_max(uR + cR, us + cs);
  }
  const double num = ((SL * hR) * (uR - SR)) - ((SR * hL) * (uL - SL));
  const double den = (hR * (uR - SR)) - (hL * (uL - SL));
  Ss = fabs(den) < 1e-14 ? 0.5 * (uL + uR) : num / den;
}

// hydrostatic_reconstruct(), kernels.hpp:126-152, as its own entry point:
// out = {left state, right state, corr_left, corr_right} (12 doubles)
__device__ __forceinline__ void reconstruct(const Cons& ul, double zl, const Cons& ur, double zr,
                                            double nx, double ny, const Phys& P, double* out) {
  const double hls = zl >= zr ? ul.h : sel_max(0.0, ul.h + (zl - zr));
  const double hrs = zr >= zl ? ur.h : sel_max(0.0, ur.h + (zr - zl));
  Cons a = ul, b = ur;
  if (!(hls == ul.h)) {
    const double vx = ul.h < P.h_dry ? 0.0 : ul.qx / ul.h, vy = ul.h < P.h_dry ? 0.0 : ul.qy / ul.h;
    a = Cons{hls, hls * vx, hls * vy};
  }
  if (!(hrs == ur.h)) {
    const double vx = ur.h < P.h_dry ? 0.0 : ur.qx / ur.h, vy = ur.h < P.h_dry ? 0.0 : ur.qy / ur.h;
    b = Cons{hrs, hrs * vx, hrs * vy};
  }
  const double pl = (0.5 * P.g) * ((ul.h * ul.h) - (hls * hls));
  const double pr = (0.5 * P.g) * ((ur.h * ur.h) - (hrs * hrs));
  const double v[12] = {a.h, a.qx, a.qy, b.h, b.qx, b.qy, 0.0, pl * nx, pl * ny, 0.0, pr * nx, pr * ny};
  for (int k = 0; k < 12; ++k) out[k] = v[k];
}

// cell_signal_speed(), kernels.hpp:167-170 (called on wet cells only).
__device__ __forceinline__ double signal_speed(const Cons& u, const Phys& P) {
  double vx, vy;
  vel(u, P.h_dry, vx, vy);
  return qsqrt(vx * vx + vy * vy) + sqrt(P.g * u.h);
}

}  // namespace swe_b200
