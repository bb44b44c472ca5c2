// swe_phys.cuh -- FP64 point physics of the explicit HLLC step, device side.
//
// Same operations, same operand order and same branch structure as the
// reference's host physics (/root/reference/proj/include/swe/kernels.hpp,
// cited per function), so the device result is bit-identical: the translation
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
// special-operand paths (the inline fast path rejects tiny numerators, so a
// zero momentum or speed would otherwise call the slow subroutine with a
// divergent warp; ncu r02: 32% of k_tile's instructions).  Results are the
// correctly rounded quotient / root in every case: for a == +-0 and finite
// non-zero b, a / b is the signed zero a * b; sqrt(+-0) = +-0.
__device__ __forceinline__ double qdiv(double a, double b) {
  const bool z = (a == 0.0) && isfinite(b) && (b != 0.0);
  const double q = (z ? 1.0 : a) / b;
  return z ? a * b : q;
}
__device__ __forceinline__ double qsqrt(double x) {
  const bool z = x == 0.0;
  const double r = sqrt(z ? 1.0 : x);
  return z ? x : r;
}

// velocity(), kernels.hpp:15-18: dry cells move with zero velocity.  The
// quotient is formed against a safe denominator so a dry (h = 0) lane never
// takes the division's special-operand slow path; the selected value is the
// reference's exactly.
__device__ __forceinline__ void vel(const Cons& u, double h_dry, double& vx, double& vy) {
  const bool dry = u.h < h_dry;
  const double hs = dry ? 1.0 : u.h;
  vx = dry ? 0.0 : qdiv(u.qx, hs);
  vy = dry ? 0.0 : qdiv(u.qy, hs);
}

// physical_flux_normal(), kernels.hpp:21-27.
__device__ __forceinline__ Flux normal_flux(const Cons& u, double nx, double ny, const Phys& P) {
  if (u.h < P.h_dry) return Flux{0.0, 0.0, 0.0};
  const double vx = qdiv(u.qx, u.h), vy = qdiv(u.qy, u.h);
  const double un = vx * nx + vy * ny;
  const double p = ((0.5 * P.g) * u.h) * u.h;
  return Flux{u.h * un, ((u.h * vx) * un) + p * nx, ((u.h * vy) * un) + p * ny};
}

// hllc_flux(), kernels.hpp:72-114, with wave_speed_estimates() (:38-66)
// inlined.  Callers guarantee non-negative depths (the reference's throw at
// :74-76 is unreachable from compute_fluxes: depths are checked first and the
// reconstruction clamps at zero).
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

  // two-rarefaction speeds, or the analytic dry-front speeds (:45-59)
  double SL, SR;
  if (dryR && !dryL) {
    const double cL = sqrt(P.g * hL);
    SL = unL - cL;
    SR = unL + 2.0 * cL;
  } else if (dryL && !dryR) {
    const double cR = sqrt(P.g * hR);
    SL = unR - 2.0 * cR;
    SR = unR + cR;
  } else {
    const double cL = sqrt(P.g * hL), cR = sqrt(P.g * hR);
    const double us = ((0.5 * (unL + unR)) + cL) - cR;
    const double cs = fabs((0.5 * (cL + cR)) + (0.25 * (unL - unR)));
    SL = sel_min(unL - cL, us - cs);
    SR = sel_max(unR + cR, us + cs);
  }
  const double aR = unR - SR, aL = unL - SL;
  const double num = ((SL * hR) * aR) - ((SR * hL) * aL);
  const double den = (hR * aR) - (hL * aL);
  const bool tiny = fabs(den) < 1e-14;
  const double Ss = tiny ? 0.5 * (unL + unR) : qdiv(num, tiny ? 1.0 : den);

  const double FL0 = hL * unL, FL1 = ((hL * unL) * unL) + (((0.5 * P.g) * hL) * hL);
  const double FR0 = hR * unR, FR1 = ((hR * unR) * unR) + (((0.5 * P.g) * hR) * hR);
  double f0, f1, ft;
  if (SL >= 0.0) {
    f0 = FL0;
    f1 = FL1;
    ft = f0 * utL;
  } else if (SR <= 0.0) {
    f0 = FR0;
    f1 = FR1;
    ft = f0 * utR;
  } else {
    const double inv = 1.0 / (SR - SL);
    const double sls = SL * SR;
    f0 = (((SR * FL0) - (SL * FR0)) + (sls * (hR - hL))) * inv;
    f1 = (((SR * FL1) - (SL * FR1)) + (sls * ((hR * unR) - (hL * unL)))) * inv;
    ft = f0 * (Ss >= 0.0 ? utL : utR);
  }
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
// {-(fmx + pr nx), -(fmy + pr ny)}; the right mass is -f0.
__device__ __forceinline__ void interior_edge(const Cons& uL, double zl, const Cons& uR, double zr,
                                              double nx, double ny, const Phys& P, double& f0,
                                              double& lx, double& ly, double& rx, double& ry) {
  // only the lower side is cut; the higher keeps its depth bitwise
  const double hls = zl >= zr ? uL.h : sel_max(0.0, uL.h + (zl - zr));
  const double hrs = zr >= zl ? uR.h : sel_max(0.0, uR.h + (zr - zl));
  Cons a = uL, b = uR;
  if (!(hls == uL.h)) {
    double vx, vy;
    vel(uL, P.h_dry, vx, vy);
    a = Cons{hls, hls * vx, hls * vy};
  }
  if (!(hrs == uR.h)) {
    double vx, vy;
    vel(uR, P.h_dry, vx, vy);
    b = Cons{hrs, hrs * vx, hrs * vy};
  }
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
  const double vx = qdiv(u.qx, u.h), vy = qdiv(u.qy, u.h);
  const double s = qsqrt(vx * vx + vy * vy);
  if (s == 0.0) return u;
  const double den = 1.0 + (((((dt * P.g) * n) * n) * s) / swe_pow43(u.h));
  return Cons{u.h, qdiv(u.qx, den), qdiv(u.qy, den)};
}

// cell_signal_speed(), kernels.hpp:167-170 (called on wet cells only).
__device__ __forceinline__ double signal_speed(const Cons& u, const Phys& P) {
  double vx, vy;
  vel(u, P.h_dry, vx, vy);
  return qsqrt(vx * vx + vy * vy) + sqrt(P.g * u.h);
}

}  // namespace swe_b200
