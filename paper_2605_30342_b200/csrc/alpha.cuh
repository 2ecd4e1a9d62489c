// alpha.cuh -- splat_alpha (R/include/gavis/raster.hpp:101-108) from a projection
// record, in fp64 with explicit FMAs: x = -q/2 with q = a dx^2 + 2b dx dy + c dy^2,
// alpha = min(o exp(x), alpha_max), 0 beyond kQSkip (fast_math.cuh). Shared by
// the VF blend (K6a) and the fp64 UA blend (K7; ua_common.cuh's pre-scaled
// ExGeo form gives the same bits: -1/2 commutes with every rounding).
#pragma once

#include "device_common.cuh"
#include "fast_math.cuh"

namespace gavis {

__device__ __forceinline__ double ex_negq(const GeoRec& r, double cxp, double cyp) {
  const double dx = cxp - r.mx, dy = cyp - r.my;
  return -0.5 * fma(dx, fma(r.ca, dx, r.cb2 * dy), r.cc * dy * dy);
}

__device__ __forceinline__ double ex_alpha(const GeoRec& r, double x, double amax) {
  const double al = (double)r.opacity * exp_neg(x);
  return x >= -0.5 * kQSkip ? (al > amax ? amax : al) : 0.0;
}

}  // namespace gavis
