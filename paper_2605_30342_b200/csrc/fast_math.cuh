// fast_math.cuh -- table-driven fp64 exp / log for the blend inner loops.
//
// libdevice's exp/log are general (overflow, NaN, denormal paths) and build
// every polynomial coefficient with two UMOVs per DFMA; in the blend loops they
// were ~115 of ~250 instructions per covered (pixel, splat) pair
// (profiles/r01_ua_blend_baseline.md). The inner loops only need
//   exp(x) for x = -q/2 in [-37.5, 0]   (q > 75 is skipped, see kQSkip)
//   ln(s)  for s in (0, 1]
// so both reduce to a 32 / 128-entry shared-memory table plus a short Taylor
// polynomial, accurate to ~1 ulp (absolute error < 3e-16 for ln).
//
// kQSkip: alpha = o*exp(-q/2) with o <= 1 and q > 75 is below 2^-54, so
// 1 - alpha rounds to exactly 1.0 and T is bit-identical whether or not the
// splat is composited; the dropped alpha*T weights are < 6e-17 each.
#pragma once

#include <cuda_runtime.h>

#include "math_tables.h"

namespace gavis {

constexpr double kQSkip = 75.0;

// Polynomial coefficients live in constant memory so each DFMA reads its
// operand straight from the constant bank (no per-use 64-bit immediate moves).
__constant__ double kExpPoly[6] = {1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0};
__constant__ double kLogPoly[7] = {1.0 / 7.0, -1.0 / 6.0, 1.0 / 5.0, -0.25, 1.0 / 3.0, -0.5, 1.0};
__constant__ double kMathConst[8] = {
    46.16624130844683,        // 0: 32 / ln2
    0.02166084939249829,      // 1: ln2/32 hi
    7.247021293269686e-19,    // 2: ln2/32 lo
    6755399441055744.0,       // 3: 1.5 * 2^52
    0.6931471805599453,       // 4: ln2 hi
    2.3190468138462996e-17,   // 5: ln2 lo
    18014398509481984.0,      // 6: 2^54
    0.0};

// Shared-memory copies of the lookup tables (namespace scope: direct shared
// addressing in the inner loops).
__shared__ double g_exp2_tab[32];
__shared__ double g_log_inv[128];
__shared__ double g_log_neg[128];

// Cooperative copy of the constant tables into shared memory (indices diverge
// per lane, which constant memory would serialise). Callers synchronise before use.
__device__ __forceinline__ void load_math_tables() {
  for (int i = threadIdx.x; i < 32 + 128 + 128; i += blockDim.x) {
    if (i < 32)
      g_exp2_tab[i] = kExp2Tab[i];
    else if (i < 160)
      g_log_inv[i - 32] = kLogInv[i - 32];
    else
      g_log_neg[i - 160] = kLogNeg[i - 160];
  }
}

// exp(x) for x in [-40, 0]: k = round(32 x / ln2), r = x - k ln2/32 (Cody-Waite
// with FMA), 2^(k/32) = 2^(k>>5) * T[k&31], e^r by a degree-6 Taylor polynomial
// (|r| <= ln2/64, remainder < 4e-18).
__device__ __forceinline__ double exp_neg(double x) {
  const double t = fma(x, kMathConst[0], kMathConst[3]);
  const int k = __double2loint(t);
  const double kd = t - kMathConst[3];
  double r = fma(kd, -kMathConst[1], x);
  r = fma(kd, -kMathConst[2], r);
  // e^r - 1 = r * (1 + r/2 + r^2/6 + r^3/24 + r^4/120 + r^5/720), Estrin's scheme
  // (dependency depth 4 instead of 6: the inner loops are fp64-latency bound)
  const double r2 = r * r;
  const double e01 = fma(r, kExpPoly[4], kExpPoly[5]);   // 1 + r/2
  const double e23 = fma(r, kExpPoly[2], kExpPoly[3]);   // 1/6 + r/24
  const double e45 = fma(r, kExpPoly[0], kExpPoly[1]);   // 1/120 + r/720
  const double e2345 = fma(r2, e45, e23);
  double p = fma(r2, e2345, e01);
  p = p * r;
  const double tj = g_exp2_tab[k & 31];
  const double res = fma(tj, p, tj);
  return __hiloint2double(__double2hiint(res) + ((k >> 5) << 20), __double2loint(res));
}

// ln(s) for finite s > 0: s = 2^e * mant, mant in [1,2); mant * inv_j = 1 + r with
// |r| < 1/256 (inv_j ~ 1/c_j from the top 7 mantissa bits), ln(1+r) by a degree-7
// Taylor polynomial, ln(s) = e ln2 - ln(inv_j) + ln(1+r).
__device__ __forceinline__ double log_pos(double s) {
  int e = 0;
  if (__double2hiint(s) < 0x00100000) {  // subnormal: scale by 2^54
    s *= kMathConst[6];
    e = -54;
  }
  const int hi = __double2hiint(s);
  e += (hi >> 20) - 1023;
  const int j = (hi >> 13) & 127;
  const double mant = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(s));
  const double r = fma(mant, g_log_inv[j], -1.0);
  // ln(1 + r) = r * (1 - r/2 + r^2/3 - r^3/4 + r^4/5 - r^5/6 + r^6/7), Estrin's scheme
  const double r2 = r * r;
  const double l01 = fma(r, kLogPoly[5], kLogPoly[6]);   // 1 - r/2
  const double l23 = fma(r, kLogPoly[3], kLogPoly[4]);   // 1/3 - r/4
  const double l45 = fma(r, kLogPoly[1], kLogPoly[2]);   // 1/5 - r/6
  const double r4 = r2 * r2;
  const double l0123 = fma(r2, l23, l01);
  const double l456 = fma(r2, kLogPoly[0], l45);          // + r^2/7
  double p = fma(r4, l456, l0123);
  p = p * r;
  const double ed = (double)e;
  return fma(ed, kMathConst[4], fma(ed, kMathConst[5], g_log_neg[j] + p));
}

}  // namespace gavis
