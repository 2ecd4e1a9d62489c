// fast_math.cuh -- table-driven fp64 exp / log for the blend inner loops.
//
// libdevice's exp/log are general (overflow, NaN, denormal paths) and build
// every polynomial coefficient with two UMOVs per DFMA; in the blend loops they
// were ~115 of ~250 instructions per covered (pixel, splat) pair
// (profiles/r01_ua_blend_baseline.md). The inner loops only need
//   exp(x) for x = -q/2 in [-37.5, 0]   (q > 75 is skipped, see kQSkip)
//   ln(s)  for s in (0, 1]
// so both reduce to a 256-entry shared-memory table plus a short Taylor
// polynomial (degree 4 / 5: the 256-entry tables halve |r| twice over the
// 32 / 128-entry tables of round 1 and drop two DFMAs from each), accurate to
// ~1 ulp (ln: absolute error < 2e-16).
//
// kQSkip: alpha = o*exp(-q/2) with o <= 1 and q > 75 is below 2^-54, so
// 1 - alpha rounds to exactly 1.0 and T is bit-identical whether or not the
// splat is composited; the dropped alpha*T weights are < 6e-17 each.
#pragma once

#include <cuda_runtime.h>

#include "math_tables.h"

namespace gavis {

constexpr double kQSkip = 75.0;
constexpr int kExpTab = 256;
constexpr int kLogTab = 256;

// Polynomial coefficients live in constant memory so each DFMA reads its
// operand straight from the constant bank (no per-use 64-bit immediate moves).
__constant__ double kExpPoly[4] = {1.0 / 24.0, 1.0 / 6.0, 0.5, 1.0};
__constant__ double kLogPoly[5] = {0.2, -0.25, 1.0 / 3.0, -0.5, 1.0};
__constant__ double kMathConst[8] = {
    369.3299304675746,        // 0: 256 / ln2
    0.0027076061740558544,    // 1: ln2/256 hi (38 significant bits: kd * hi is exact)
    6.432011555819173e-15,    // 2: ln2/256 lo
    6755399441055744.0,       // 3: 1.5 * 2^52
    0.6931471805599453,       // 4: ln2 (correctly rounded)
    0.0,                      // 5: (unused)
    18014398509481984.0,      // 6: 2^54
    0.0};

// Shared-memory copies of the lookup tables (namespace scope: direct shared
// addressing in the inner loops).
// The two log tables interleaved as {1/c_j, -ln(1/c_j)} pairs: one 128-bit load
// per lookup instead of two 64-bit ones (GAVIS_LOG_PAIR=1; A/B).
#ifndef GAVIS_LOG_PAIR
#define GAVIS_LOG_PAIR 1
#endif
__shared__ double g_exp2_tab[kExpTab];
#if GAVIS_LOG_PAIR
__shared__ double2 g_log_tab[kLogTab];
#else
__shared__ double g_log_inv[kLogTab];
__shared__ double g_log_neg[kLogTab];
#endif

// Cooperative copy of the constant tables into shared memory (indices diverge
// per lane, which constant memory would serialise). Callers synchronise before use.
__device__ __forceinline__ void load_math_tables() {
  for (int i = threadIdx.x; i < kExpTab + kLogTab; i += blockDim.x) {
    if (i < kExpTab)
      g_exp2_tab[i] = kExp2Tab[i];
    else
#if GAVIS_LOG_PAIR
      g_log_tab[i - kExpTab] = make_double2(kLogInv[i - kExpTab], kLogNeg[i - kExpTab]);
#else
      g_log_inv[i - kExpTab] = kLogInv[i - kExpTab], g_log_neg[i - kExpTab] = kLogNeg[i - kExpTab];
#endif
  }
}

// exp(x) for x in [-40, 0]: k = round(256 x / ln2), r = x - k ln2/256 (Cody-Waite
// with FMA), 2^(k/256) = 2^(k>>8) * T[k&255], e^r - 1 by a degree-4 Taylor
// polynomial (|r| <= ln2/512: remainder < 4e-17 relative). Inputs below -40 give
// unspecified finite/NaN values; callers discard them (kQSkip).
__device__ __forceinline__ double exp_neg(double x) {
  const double t = fma(x, kMathConst[0], kMathConst[3]);
  const int k = __double2loint(t);
  const double kd = t - kMathConst[3];
  double r = fma(kd, -kMathConst[1], x);
  r = fma(kd, -kMathConst[2], r);
  // e^r - 1 = r * (1 + r/2 + r^2/6 + r^3/24), Estrin's scheme (depth 3)
  const double r2 = r * r;
  const double e01 = fma(r, kExpPoly[2], kExpPoly[3]);   // 1 + r/2
  const double e23 = fma(r, kExpPoly[0], kExpPoly[1]);   // 1/6 + r/24
  const double p = fma(r2, e23, e01) * r;
  const double tj = g_exp2_tab[k & (kExpTab - 1)];
  const double res = fma(tj, p, tj);
  return __hiloint2double(__double2hiint(res) + ((k >> 8) << 20), __double2loint(res));
}

// ln(s) for finite s > 0 (log_pos), and for the per-entry entropy terms
// s (hl + C_H - ln s) of the blends (log_blend): there s = 0 must give a finite
// value (s * finite = +0 exactly) and a subnormal s may get a wrong but finite
// one -- the term is then below 1e-305 either way -- so log_blend skips
// log_pos's subnormal rescaling (4 instructions per composited entry).
// s = 2^e * mant, mant in [1,2); mant * inv_j = 1 + r with
// |r| < 1/512 (inv_j ~ 1/c_j from the top 8 mantissa bits), ln(1+r) by a degree-5
// Taylor polynomial (remainder < 1e-17), ln(s) = e ln2 - ln(inv_j) + ln(1+r).
template <bool SUBNORMAL>
__device__ __forceinline__ double log_table(double s) {
  int e = 0;
  if (SUBNORMAL && __double2hiint(s) < 0x00100000) {  // subnormal: scale by 2^54
    s *= kMathConst[6];
    e = -54;
  }
  const int hi = __double2hiint(s);
  e += (hi >> 20) - 1023;
  const int j = (hi >> 12) & (kLogTab - 1);
  const double mant = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, __double2loint(s));
#if GAVIS_LOG_PAIR
  const double2 tab = g_log_tab[j];
#else
  const double2 tab = make_double2(g_log_inv[j], g_log_neg[j]);
#endif
  const double r = fma(mant, tab.x, -1.0);
  // ln(1 + r) = r * (1 - r/2 + r^2/3 - r^3/4 + r^4/5), Estrin's scheme
  const double r2 = r * r;
  const double l01 = fma(r, kLogPoly[3], kLogPoly[4]);   // 1 - r/2
  const double l23 = fma(r, kLogPoly[1], kLogPoly[2]);   // 1/3 - r/4
  const double l234 = fma(r2, kLogPoly[0], l23);         // + r^2/5
  const double p = fma(r2, l234, l01) * r;
  return fma((double)e, kMathConst[4], tab.y + p);
}

__device__ __forceinline__ double log_pos(double s) { return log_table<true>(s); }
__device__ __forceinline__ double log_blend(double s) { return log_table<false>(s); }

}  // namespace gavis
