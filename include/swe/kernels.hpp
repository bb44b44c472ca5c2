// swe/kernels.hpp -- the point-physics entry points of the reference's
// kernels.hpp (reference include/swe/kernels.hpp:15-216) for callers that use
// them directly (its io.hpp VTK writer, its own kernel-level tests
// tests/test_kernels.cpp, which compile unchanged against this header).
//
// velocity() is the reference's two-line output helper (kernels.hpp:15-18),
// kept on the host for post-processing.  The fluxes and the friction
// evaluate on the DEVICE through swe_dev_point_eval (the same __device__
// functions the step kernels use, csrc/swe_phys.cuh) -- there is no host
// implementation of the step's physics.  Each call is a round trip to the
// GPU: meant for tests and diagnostics, not for loops.
#pragma once

#include <cmath>
#include <limits>
#include <span>
#include <string>

#include "swe/core.hpp"
#include "swe_dev.h"

namespace swe {

// kernels.hpp:15-18
inline Vec2 velocity(const ConservedState& u, double h_dry) {
  if (u.h < h_dry) return {0.0, 0.0};
  return {u.qx / u.h, u.qy / u.h};
}

namespace detail {
inline swe_params to_params(const PhysParams& p) { return {p.g, p.h_dry, p.cfl, p.dt_max, p.h_ref}; }

inline void point_eval(int kind, const double* l, const double* r, const double* z,
                       const double* n, double* out, const PhysParams& p) {
  const swe_params sp = to_params(p);
  if (swe_dev_point_eval(kind, 1, &sp, l, r, z, n, out) != SWE_OK)
    throw error(std::string("point evaluation on the device failed: ") + swe_dev_last_error());
}
}  // namespace detail

// kernels.hpp:21-27
inline Flux3 physical_flux_normal(const ConservedState& u, Vec2 n, const PhysParams& p) {
  const double l[3] = {u.h, u.qx, u.qy}, nn[2] = {n.x, n.y};
  double out[3];
  detail::point_eval(5, l, nullptr, nullptr, nn, out, p);
  return {out[0], out[1], out[2]};
}

/// kernels.hpp:33-37
struct WaveSpeeds {
  double SL = 0.0;
  double Sstar = 0.0;
  double SR = 0.0;
};

// kernels.hpp:38-66
inline WaveSpeeds wave_speed_estimates(double hL, double uL, double hR, double uR,
                                       const PhysParams& p) {
  const double l[3] = {hL, uL, 0.0}, r[3] = {hR, uR, 0.0};
  double out[3];
  detail::point_eval(6, l, r, nullptr, nullptr, out, p);
  return {out[0], out[1], out[2]};
}

// kernels.hpp:72-114
inline Flux3 hllc_flux(const ConservedState& left, const ConservedState& right, Vec2 n,
                       const PhysParams& p) {
  if (left.h < 0.0 || right.h < 0.0)
    throw numeric_error("hllc_flux: negative depth (hL=" + std::to_string(left.h) +
                        ", hR=" + std::to_string(right.h) + ")");
  const double l[3] = {left.h, left.qx, left.qy}, r[3] = {right.h, right.qx, right.qy};
  const double nn[2] = {n.x, n.y};
  double out[3];
  detail::point_eval(0, l, r, nullptr, nn, out, p);
  return {out[0], out[1], out[2]};
}

/// kernels.hpp:121-124
struct ReconstructedInterface {
  ConservedState left, right;
  Flux3 corr_left, corr_right;
};

// kernels.hpp:126-152
inline ReconstructedInterface hydrostatic_reconstruct(const ConservedState& ul, double zl,
                                                      const ConservedState& ur, double zr,
                                                      Vec2 n, const PhysParams& p) {
  const double l[3] = {ul.h, ul.qx, ul.qy}, r[3] = {ur.h, ur.qx, ur.qy}, z[2] = {zl, zr};
  const double nn[2] = {n.x, n.y};
  double o[12];
  detail::point_eval(7, l, r, z, nn, o, p);
  return {{o[0], o[1], o[2]}, {o[3], o[4], o[5]}, {o[6], o[7], o[8]}, {o[9], o[10], o[11]}};
}

// kernels.hpp:156-164
inline Flux3 wall_flux(const ConservedState& u, Vec2 n, const PhysParams& p) {
  const double l[3] = {u.h, u.qx, u.qy}, nn[2] = {n.x, n.y};
  double out[3];
  detail::point_eval(1, l, nullptr, nullptr, nn, out, p);
  return {out[0], out[1], out[2]};
}

// kernels.hpp:167-170
inline double cell_signal_speed(const ConservedState& u, const PhysParams& p) {
  const double l[3] = {u.h, u.qx, u.qy};
  double out[1];
  detail::point_eval(8, l, nullptr, nullptr, nullptr, out, p);
  return out[0];
}

// kernels.hpp:174-186: the min-reduction runs on the device (swe_dev_stable_dt)
inline double stable_dt(std::span<const double> h, std::span<const double> qx,
                        std::span<const double> qy, std::span<const double> inradius,
                        const PhysParams& p) {
  const swe_params sp = detail::to_params(p);
  double dt = 0.0;
  long long bad = -1;
  const int rc = swe_dev_stable_dt(0, static_cast<long long>(h.size()), &sp, h.data(), qx.data(),
                                   qy.data(), inradius.data(), &dt, &bad);
  if (rc == SWE_NONFINITE_SPEED)
    throw numeric_error("stable_dt: non-finite velocity in cell " + std::to_string(bad));
  if (rc != SWE_OK)
    throw error(std::string("stable_dt on the device failed: ") + swe_dev_last_error());
  return dt;
}

// kernels.hpp:191-199
inline ConservedState apply_friction(const ConservedState& u, double n_manning, double dt,
                                     const PhysParams& p) {
  const double l[3] = {u.h, u.qx, u.qy}, z[2] = {n_manning, dt};
  double out[3];
  detail::point_eval(3, l, nullptr, z, nullptr, out, p);
  return {out[0], out[1], out[2]};
}

// kernels.hpp:205-216
inline ConservedState clamp_dry(const ConservedState& u, const PhysParams& p,
                                double* clipped_depth = nullptr) {
  const double l[3] = {u.h, u.qx, u.qy};
  double out[5];
  detail::point_eval(9, l, nullptr, nullptr, nullptr, out, p);
  if (out[4] != 0.0)
    throw numeric_error("clamp_dry: depth " + std::to_string(u.h) +
                        " below the positivity tolerance");
  if (clipped_depth && out[3] != 0.0) *clipped_depth += out[3];
  return {out[0], out[1], out[2]};
}

}  // namespace swe
