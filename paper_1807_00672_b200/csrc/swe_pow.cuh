// swe_pow.cuh -- h^(4/3) for the Manning friction denominator
// (kernels.hpp:197, std::pow(u.h, 4.0 / 3.0)).
#pragma once

namespace swe_b200 {

__device__ __forceinline__ double swe_pow43(double h) { return pow(h, 4.0 / 3.0); }

}  // namespace swe_b200
