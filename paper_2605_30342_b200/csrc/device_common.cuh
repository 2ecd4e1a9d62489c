// device_common.cuh -- records, camera block and fp64 math shared by the kernels.
//
// Every expression that feeds a discrete decision of the reference (culling,
// tile rectangles, coverage, alpha, transmittance, early termination) is
// written with the reference's operation order and compiled with -fmad=false,
// so it rounds exactly like the reference's double code
// (R/include/gavis/raster.hpp:51-108, vfield.hpp:96-112, uncertainty.hpp:55-59).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace gavis {

constexpr double kY00 = 0.28209479177387814;        // sh.hpp:28
constexpr double kGaussEntropy = 4.256815599614018;  // uncertainty.hpp:19
constexpr int kMaxFieldDegree = 4;                   // device instantiations (registers)
constexpr int kMaxFieldDegreeRT = 20;                // runtime-degree path (local memory), construct_field's limit
constexpr int kDegRT = 99;                            // template tag of the runtime-degree path
constexpr int kMaxColorDegree = 3;

// Per-view camera block, precomputed on the host with the reference's own
// formulas (CameraView::focal_x etc., model.hpp:75-78; Jacobian limits
// raster.hpp:60-61) so the transcendental tan() is evaluated once, by libm.
struct DevCam {
  double R[9];      // row-major camera-to-world
  double pos[3];
  double fx, fy, cx, cy, limx, limy, near_plane;
  int32_t width, height, tiles_x, tiles_y;
  int64_t tile_base;  // first global tile id of this view inside the batch
  int64_t pix_base;   // first output pixel of this view
};

// One projected splat (ImageSpaceSplat, raster.hpp:37-44) in 64 bytes, in the
// form the blends consume it (no per-use decoding): the conic pre-scaled by -1/2
// (a power of two: exact), so x = -q/2 comes out of two FMAs; the opacity
// widened once; the exact coverage interval per axis as (start, width).
struct __align__(16) GeoRec {
  double mx, my;        // mean
  double na, nb, nc;    // -a/2, -b, -c/2 of the conic (a, b, c)
  double o;             // opacity
  double depth;         // NaN marks a culled slot (debug dumps only)
  int32_t cov_x;        // x0 | (x1 - x0) << 16 : pixels with |x+0.5-mx| <= r
  int32_t cov_y;        // y0 | (y1 - y0) << 16; kCovEmpty when none
};
constexpr int32_t kCovEmpty = 0xFFFF;  // start 65535, width 0: never hit (widths < 65535)

// Entropy-track constants of one splat (compensated_alpha, uncertainty.hpp:55-59):
// alpha* = A*alpha + B with A = v + beta(1-v), B = o0(1-beta)(1-v); hl is the
// splat's 1/2 log|Q_c| (constant provider: 3 ln sigma_c; sh_propagation:
// 1/2 sum_c ln q_c(d), uncertainty.hpp:143-163).
// omv = 1 - v and hlc = hl + C_H are stored too (the blends read them per
// pixel); 48 bytes: a multiple of 16 for cp.async / bulk copies.
struct __align__(16) UaRec {
  double A, B, v, omv, hlc, hl;
};

__device__ __forceinline__ int cov_lo(int32_t packed) { return packed & 0xFFFF; }
__device__ __forceinline__ int cov_width(int32_t packed) { return (int)((uint32_t)packed >> 16); }

// Coverage rectangle as (x0, x1-x0, y0, y1-y0) for a two-compare unsigned test
// (unsigned)(px - x0) <= x1 - x0; an empty axis is (65535, 0), never hit.
__device__ __forceinline__ int4 cover_rect4(int32_t cov_x, int32_t cov_y) {
  return make_int4(cov_lo(cov_x), cov_width(cov_x), cov_lo(cov_y), cov_width(cov_y));
}

__device__ __forceinline__ bool in_rect4(int4 r, int px, int py) {
  return (unsigned)(px - r.x) <= (unsigned)r.y && (unsigned)(py - r.z) <= (unsigned)r.w;
}

// eval_real_sh_block (sh.hpp:38-79), fixed maximum degree, same recurrence and
// operation order.
template <int DEG>
__device__ __forceinline__ void eval_sh(double x, double y, double z, double* out) {
  const double s = sqrt(x * x + y * y);
  const double cphi = s > 1e-14 ? x / s : 1.0;
  const double sphi = s > 1e-14 ? y / s : 0.0;
  const double kSqrt2 = 1.4142135623730951;
  double pmm = kY00;
  double cm = 1.0, sm = 0.0;
#pragma unroll
  for (int m = 0; m <= DEG; ++m) {
    if (m > 0) {
      pmm *= s * sqrt((2.0 * m + 1.0) / (2.0 * m));
      double cnext = cm * cphi - sm * sphi;
      sm = sm * cphi + cm * sphi;
      cm = cnext;
    }
    double plm = pmm, plm_prev = 0.0;
#pragma unroll
    for (int l = m; l <= DEG; ++l) {
      if (l > m) {
        double next;
        if (l == m + 1) {
          next = z * sqrt(2.0 * m + 3.0) * pmm;
        } else {
          double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
          double b = sqrt(((double)(l - 1) * (l - 1) - (double)m * m) /
                          (4.0 * (double)(l - 1) * (l - 1) - 1.0));
          next = a * (z * plm - b * plm_prev);
        }
        plm_prev = plm;
        plm = next;
      }
      if (m == 0) {
        out[l * l + l] = plm;
      } else {
        out[l * l + l + m] = kSqrt2 * plm * cm;
        out[l * l + l - m] = kSqrt2 * plm * sm;
      }
    }
  }
}

// Runtime-degree variant (any degree; `out` holds (degree + 1)^2 values): the
// variance-propagation provider and fields above degree 4.
__device__ __forceinline__ void eval_sh_rt(int degree, double x, double y, double z, double* out) {
  const double s = sqrt(x * x + y * y);
  const double cphi = s > 1e-14 ? x / s : 1.0;
  const double sphi = s > 1e-14 ? y / s : 0.0;
  const double kSqrt2 = 1.4142135623730951;
  double pmm = kY00;
  double cm = 1.0, sm = 0.0;
  for (int m = 0; m <= degree; ++m) {
    if (m > 0) {
      pmm *= s * sqrt((2.0 * m + 1.0) / (2.0 * m));
      double cnext = cm * cphi - sm * sphi;
      sm = sm * cphi + cm * sphi;
      cm = cnext;
    }
    double plm = pmm, plm_prev = 0.0;
    for (int l = m; l <= degree; ++l) {
      if (l > m) {
        double next;
        if (l == m + 1) {
          next = z * sqrt(2.0 * m + 3.0) * pmm;
        } else {
          double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
          double b = sqrt(((double)(l - 1) * (l - 1) - (double)m * m) /
                          (4.0 * (double)(l - 1) * (l - 1) - 1.0));
          next = a * (z * plm - b * plm_prev);
        }
        plm_prev = plm;
        plm = next;
      }
      if (m == 0) {
        out[l * l + l] = plm;
      } else {
        out[l * l + l + m] = kSqrt2 * plm * cm;
        out[l * l + l - m] = kSqrt2 * plm * sm;
      }
    }
  }
}

// covered_pixel_range (raster.hpp:138-141).
__device__ __forceinline__ void covered_pixel_range(double m, double r, int n, int& lo, int& hi) {
  int a = (int)ceil(m - r - 0.5);
  int b = (int)floor(m + r - 0.5);
  lo = a > 0 ? a : 0;
  hi = b < n - 1 ? b : n - 1;
}

// splat_covers (raster.hpp:97-99) along one axis.
__device__ __forceinline__ bool covers_1d(int x, double m, double r) {
  return fabs((x + 0.5) - m) <= r;
}

// Exact pixel interval of splat_covers along one axis, starting from the
// binning interval [lo, hi] (never more than a pixel away).
__device__ __forceinline__ int32_t exact_cover(int lo, int hi, int n, double m, double r) {
  if (lo > hi) return kCovEmpty;
  while (lo > 0 && covers_1d(lo - 1, m, r)) --lo;
  while (lo <= hi && !covers_1d(lo, m, r)) ++lo;
  while (hi < n - 1 && covers_1d(hi + 1, m, r)) ++hi;
  while (hi >= lo && !covers_1d(hi, m, r)) --hi;
  if (lo > hi) return kCovEmpty;
  return (int32_t)(lo | ((hi - lo) << 16));
}

}  // namespace gavis
