// swe/kernels.hpp -- the point-physics entry points of the reference's
// kernels.hpp (reference include/swe/kernels.hpp:15-216) for callers that use
// them directly (its io.hpp VTK writer, kernel-level tests).
//
// velocity() is the reference's two-line output helper (kernels.hpp:15-18),
// kept on the host for post-processing.  The fluxes and the friction
// evaluate on the DEVICE through swe_dev_point_eval (the same __device__
// functions the step kernels use, csrc/swe_phys.cuh) -- there is no host
// implementation of the step's physics.  Each call is a round trip to the
// GPU: meant for tests and diagnostics, not for loops.
#pragma once

#include <cmath>
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

// kernels.hpp:156-164
inline Flux3 wall_flux(const ConservedState& u, Vec2 n, const PhysParams& p) {
  const double l[3] = {u.h, u.qx, u.qy}, nn[2] = {n.x, n.y};
  double out[3];
  detail::point_eval(1, l, nullptr, nullptr, nn, out, p);
  return {out[0], out[1], out[2]};
}

// kernels.hpp:191-199
inline ConservedState apply_friction(const ConservedState& u, double n_manning, double dt,
                                     const PhysParams& p) {
  const double l[3] = {u.h, u.qx, u.qy}, z[2] = {n_manning, dt};
  double out[3];
  detail::point_eval(3, l, nullptr, z, nullptr, out, p);
  return {out[0], out[1], out[2]};
}

}  // namespace swe
