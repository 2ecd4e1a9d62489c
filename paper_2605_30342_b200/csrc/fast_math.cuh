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
  double p = fma(r, kExpPoly[0], kExpPoly[1]);
  p = fma(p, r, kExpPoly[2]);
  p = fma(p, r, kExpPoly[3]);
  p = fma(p, r, kExpPoly[4]);
  p = fma(p, r, kExpPoly[5]);
  p = p * r;  // e^r - 1
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
  double p = fma(r, kLogPoly[0], kLogPoly[1]);
  p = fma(p, r, kLogPoly[2]);
  p = fma(p, r, kLogPoly[3]);
  p = fma(p, r, kLogPoly[4]);
  p = fma(p, r, kLogPoly[5]);
  p = fma(p, r, kLogPoly[6]);
  p = p * r;  // ln(1 + r)
  const double ed = (double)e;
  return fma(ed, kMathConst[4], fma(ed, kMathConst[5], g_log_neg[j] + p));
}

}  // namespace gavis
