// alpha.cuh -- splat_alpha (R/include/gavis/raster.hpp:101-108) from a projection
// record, in fp64 with explicit FMAs: x = -q/2 with q = a dx^2 + 2b dx dy + c dy^2,
// alpha = min(o exp(x), alpha_max), 0 beyond kQSkip (fast_math.cuh). Shared by
// the VF blend (K6a) and the fp64 UA blend (K7); the record carries the conic
// pre-scaled by -1/2 (device_common.cuh), which gives the same bits as scaling
// q: -1/2 commutes with every rounding.
#pragma once

#include "device_common.cuh"
#include "fast_math.cuh"

namespace gavis {

// x = -q/2 at the pixel centre, q = a dx^2 + 2b dx dy + c dy^2, from the
// pre-scaled conic (-a/2, -b, -c/2): the same bits as -0.5 * q.
__device__ __forceinline__ double ex_negq(const GeoRec& r, double cxp, double cyp) {
  const double dx = cxp - r.mx, dy = cyp - r.my;
  return fma(dx, fma(r.na, dx, r.nb * dy), r.nc * dy * dy);
}

// alpha = min(o exp(-q/2), alpha_max); q > kQSkip -> 0 (T bit-identical, fast_math.cuh).
__device__ __forceinline__ double ex_alpha(const GeoRec& r, double x, double amax) {
  const double al = r.o * exp_neg(x);
  return x >= -0.5 * kQSkip ? (al > amax ? amax : al) : 0.0;
}

}  // namespace gavis
