// kernels_ua_fast.cu -- the UA blends on 16x16 tiles with the tensor-core colour:
// the default fp64 blend (K7, ua_blend_exact_mma_kernel, and its opt-in TMA-ring
// form), the certified fp32 blend (K7f), its fp64 redo (K7r), and the image score
// (K8).
//
// K7f computes the same two tracks as the exact fp64 kernels (ua_common.cuh;
// rasterize raster.hpp:191-229 and render_entropy_core uncertainty.hpp:177-236)
// in fp32, except for the quadratic form q, which stays fp64 (a thin splat's
// conic is ill-conditioned: q cancels in fp32). exp and ln run on the SFU
// (ex2/lg2.approx). The only discrete decision of the loop that fp32 can get
// wrong is early termination (T < cutoff; coverage is integer and exact), so
// the kernel carries an error bound for each transmittance and flags a pixel
// when a termination test it made was closer to the cutoff than that bound.
// Flagged pixels are recomputed with the exact fp64 steps by K7r; every other
// pixel's stop point -- hence contributor counts -- is that of the fp64
// reference.
//
// Error bound (relative, T_fp32 vs T_fp64, u = 2^-24). A composited entry
// multiplies T by (1 - a). fp32 perturbs a by |da| <= a (1.5 q + 8) u (q -> fp32
// and the ln2 scaling 1.5 q u, ex2.approx <= 4u, products and the A/B/v
// roundings of a* <= 4u), so the new T = fma(-T, a, T) (one rounding) is off by
// |da| / (1 - a) + u. On the splat's support q <= 2 ln(o/a), hence
//   a < 1/2 :  a (1.5 q + 8) / (1 - a) <= 2 (3/e + 8 a)   <= 2.2 + 16 a/(1-a)
//   a >= 1/2:  q <= 2 ln 2, a (1.5 q + 8) / (1 - a)        <= 10.1 a/(1-a)
// and for a* = clamp(A a + B): [A a (1.5 q + 8) + 3 a*] / (1 - a*) <= 2.2 +
// 22 a*/(1-a*) (A a (1.5 q + 8) <= 8 A o <= 16 a* when a* >= 1/2). After k
// entries, with S = sum a/(1-a) over them, the relative error is at most
//   u (22 S + 3.2 k + 16).
// A second bound splits the steps at a = e^-10 instead of 1/2: above it
// q <= 20 gives a (1.5 q + 8)/(1 - a) <= 38 a/(1-a) (41 for a*), below it the
// term is < 2e-3 (< 4e-3 for a*), so the error is also <= u (41 S + 1.004 k + 16);
// the window uses the smaller (deep pixels: many steps, few of them opaque).
// The kernel accumulates S per track (one rcp.approx + one FMA per entry) and
// flags a pixel when min |T/cutoff - 1| over the two tests bracketing its stop
// (or its final T, if it never stops) is within twice that bound
// (cert_base + cert_per_step k + cert_sum S, from the host).
#include "ua_common.cuh"

#include <cuda_fp16.h>
#include <cstdlib>

namespace gavis {

namespace {

constexpr int kFastBatch = 192;
#ifndef GAVIS_FAST_MIN_BLOCKS
#define GAVIS_FAST_MIN_BLOCKS 3
#define GAVIS_FAST_BATCH_MMA 128
#endif
// 3 CTAs per SM (80 registers) of 128-entry batches; 4 CTAs (64 registers, 40 B
// of spills) of 64-entry batches measured 2018 vs 2031 views/s at config 3
constexpr int kFastMinBlocks = GAVIS_FAST_MIN_BLOCKS;
constexpr int kFastBatchMma = GAVIS_FAST_BATCH_MMA;
constexpr float kNegHalfLog2e = -0.72134752044448170f;  // -0.5 / ln 2
constexpr float kLn2f = 0.69314718055994531f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// One staged splat: fp64 mean/conic for q, fp32 opacity and depth.
struct __align__(16) FGeo {
  double mx, my, ca, cb2, cc;
  float o, depth;
};

// Colour of a (pixel, entry) pair, clamp(sum_i c_i Y_i(ray), 0, 1) per channel
// (model.hpp:49-62), two ways:
//  * FFMA: fp32 coefficient rows staged per entry, packed fp32x2 FMAs per pixel
//    against the pixel's SH basis (48 MACs per pair at degree 3);
//  * MMA (default): per group of 8 hit entries the warp computes the 32 x 24
//    colour block [pixels x (entry, channel)] = Y[32 x 16] C[16 x 24] on the
//    tensor cores with mma.sync m16n8k16 in split fp16 (x = hi + lo, products
//    hi*hi + hi*lo + lo*hi accumulated in fp32: ~22-bit operands, colour error
//    ~1e-6), then transposes it through shared memory so each lane reads its
//    own pixel's colours. Coefficients are split once per scene
//    (SceneDev::colors_split) and staged as-is.
constexpr int kColWords = 52;  // per staged entry: hi [3][16] f16 (24 words), lo (24), pad (4)
// The warp's colour block: 32 pixel rows of [channel][8 entries] floats. The
// padded stride 26 keeps the per-pixel reads (LDS.64, lane = row) conflict-free;
// the mma fragment stores (STS.64) then see 2-way conflicts. An XOR swizzle of
// the entry pairs (stride 24, GAVIS_TR_SWIZZLE=1) removes those too (store
// conflicts 198 M -> 33 M per 16 views) but costs an index op per access and was
// 2 % slower overall: the shared-memory pipe is not the limiter.
#ifndef GAVIS_TR_SWIZZLE
#define GAVIS_TR_SWIZZLE 0
#endif
#if GAVIS_TR_SWIZZLE
constexpr int kTrStride = 24;
__device__ __forceinline__ int tr_idx(int row, int col) { return row * kTrStride + (col ^ (((row >> 2) & 3) << 1)); }
#else
constexpr int kTrStride = 26;
__device__ __forceinline__ int tr_idx(int row, int col) { return row * kTrStride + col; }
#endif

template <int LC, bool RGB, bool ENT, bool MMA>
struct FStage {
  static constexpr size_t col_bytes() {
    return MMA ? sizeof(uint32_t) * kColWords : sizeof(float) * Col<LC>::STRIDE;
  }
  static constexpr size_t tr_bytes() { return (RGB && MMA) ? 8 * 32 * kTrStride * sizeof(float) : 0; }
  static constexpr size_t bytes(int batch) {
    return (size_t)batch * (sizeof(FGeo) + sizeof(int4) + (ENT ? sizeof(float4) : 0) +
                            (RGB ? col_bytes() : 0)) + tr_bytes();
  }
};

__device__ __forceinline__ uint32_t pack_half2(float x, float y) {
  const __half2 h = __floats2half2_rn(x, y);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// x = hi + lo with hi, lo fp16 (lo rounds the exact fp32 residual)
__device__ __forceinline__ void split_half2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 f = __half22float2(h);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = pack_half2(x - f.x, y - f.y);
}

__device__ __forceinline__ void hmma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                          uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Per (particle, channel, 4 coefficients): the hi/lo fp16 words of the staged
// colour record ([hi: ch][8] [lo: ch][8] [pad 4], 52 words), as fstage_batch
// stages them; coefficients past NB are 0.
template <int LC>
__device__ __forceinline__ void split_colour_quad(const float* colors, int64_t g, int ch, int q,
                                                  uint32_t* rec) {
  constexpr int NB = Col<LC>::NB, NBP = Col<LC>::NBP, CS = Col<LC>::STRIDE;
  const float* src = colors + g * CS + ch * NBP;
  float x[4];
  if (NB == 16) {
    const float4 v4 = __ldg(reinterpret_cast<const float4*>(src) + q);
    x[0] = v4.x;
    x[1] = v4.y;
    x[2] = v4.z;
    x[3] = v4.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = (4 * q + i < NB) ? __ldg(src + 4 * q + i) : 0.f;
  }
  uint32_t h0, l0, h1, l1;
  split_half2(x[0], x[1], h0, l0);
  split_half2(x[2], x[3], h1, l1);
  uint32_t* dst = rec + ch * 8 + 2 * q;
  *reinterpret_cast<uint2*>(dst) = make_uint2(h0, h1);
  *reinterpret_cast<uint2*>(dst + 24) = make_uint2(l0, l1);
}

// Builds SceneDev::colors_split: one thread per (particle, channel, quad); the
// padding words are zeroed by the (ch, q) = (0, 0) thread.
template <int LC>
__global__ void split_colors_kernel(const float* colors, int64_t n, uint32_t* out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n * 12) return;
  const int64_t g = k / 12;
  const int r = (int)(k - g * 12), ch = r >> 2, q = r & 3;
  uint32_t* rec = out + g * kColWords;
  split_colour_quad<LC>(colors, g, ch, q, rec);
  if (r == 0) *reinterpret_cast<uint4*>(rec + 48) = make_uint4(0u, 0u, 0u, 0u);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Stage entries [base, base+n) of the tile list: the fp32 forms are computed
// once here, per tile, not per pixel. With the tensor-core colour path the
// colours come pre-split (SceneDev::colors_split): threads [0, 128) stage the
// geometry, threads [128, 256) copy the colour records with cp.async (13
// independent 16-byte copies per entry in flight, no register round trip).
template <int LC, bool RGB, bool ENT, bool MMA>
__device__ __forceinline__ void fstage_batch(const UaBlendArgs& a, const GeoRec* geo,
                                             const UaRec* uar, uint32_t base, int n, FGeo* s_geo,
                                             int4* s_rect, float4* s_ua, void* s_col) {
  constexpr int CS = Col<LC>::STRIDE;
  constexpr int V4 = CS / 4;
  constexpr int kHalf = 128;
  if (RGB && MMA) {
    const int t = threadIdx.x;
    if (t >= kHalf) {
      uint4* dst = reinterpret_cast<uint4*>(s_col);
      for (int j = t - kHalf; j < n; j += kHalf) {
        const uint4* src = a.scene.colors_split + (int64_t)a.vals[base + j] * (kColWords / 4);
#pragma unroll
        for (int w = 0; w < kColWords / 4; ++w) cp_async16(dst + j * (kColWords / 4) + w, src + w);
      }
      cp_async_wait_all();
      return;
    }
  }
  const int t0 = threadIdx.x, nt = (RGB && MMA) ? kHalf : blockDim.x;
  for (int j = t0; j < n; j += nt) {
    const uint32_t g = a.vals[base + j];
    const GeoRec r = geo[g];
    FGeo f;
    f.mx = r.mx;
    f.my = r.my;
    f.ca = -2.0 * r.na;  // a, 2b, c: exact rescaling of the K1 record
    f.cb2 = -2.0 * r.nb;
    f.cc = -2.0 * r.nc;
    f.o = (float)r.o;  // widened from the scene's fp32 opacity: exact
    f.depth = (float)r.depth;
    s_geo[j] = f;
    s_rect[j] = cover_rect4(r.cov_x, r.cov_y);
    if (ENT) {
      const UaRec u = uar[g];
      s_ua[j] = make_float4((float)u.A, (float)u.B, (float)u.v, (float)u.hlc);
    }
  }
  if (RGB && !MMA) {
    const float4* colors4 = reinterpret_cast<const float4*>(a.scene.colors);
    for (int k = threadIdx.x; k < n * V4; k += blockDim.x) {
      const int j = k / V4, qd = k - j * V4;
      const uint32_t g = a.vals[base + j];
      reinterpret_cast<float4*>(s_col)[k] = __ldg(colors4 + (int64_t)g * V4 + qd);
    }
  }
}

template <int LC>
struct FPix {
  // fp32 running state; the sums are folded into fp64 after every 32-entry chunk
  float T, Tp, r0, r1, r2, dp;
  float Te, Tep, h, w0, ed;
  float S, Se;  // sum a/(1-a) over composited entries, per track (error bound)
  double R0, R1, R2, DP, H, W0, ED;
  int n_rgb, n_ent;
  bool rd, edn;
};

template <int LC, bool EXTRA>
__device__ __forceinline__ void fold(FPix<LC>& P) {
  P.R0 += (double)P.r0;
  P.R1 += (double)P.r1;
  P.R2 += (double)P.r2;
  P.H += (double)P.h;
  P.W0 += (double)P.w0;
  P.r0 = P.r1 = P.r2 = P.h = P.w0 = 0.f;
  if (EXTRA) {
    P.DP += (double)P.dp;
    P.ED += (double)P.ed;
    P.dp = P.ed = 0.f;
  }
}

// The certification window of a track after k composited entries with
// S = sum a/(1-a): the smaller of the two bounds (header; twice each).
__device__ __forceinline__ float cert_window_of(const UaBlendArgs& a, float k, float S) {
  return a.cert_base + fminf(fmaf(a.cert_per_step, k, a.cert_sum * S),
                             fmaf(a.cert_per_step2, k, a.cert_sum2 * S));
}

// Score bound: a rigorous bound on |H_fp32 - H_fp64| of one pixel's entropy
// (the certified select_nbv widens its fp64 re-scoring window by the folded
// bounds of the best and of each candidate, so its argmax is the fp64 one).
// Per composited entry the entropy term is s (c - ln s), s = a* T* v, with one
// c = 3 ln sigma_c + C_H for every entry (constant provider). With u = 2^-24:
//  * T* is within eps_T = u (22 S + 3.2 k + 16) (relative; the stop-test bound
//    above, half the certification window) for every k;
//  * |da*| <= [A a (1.5 q + 8) + 3 a*] u with A a <= a*: <= 41 u a* for
//    q <= 20, and A a (1.5 q + 8) <= o e^-10 38 <= 1.7e-3 o for q > 20;
//  * so |ds| <= s (eps_T + 43 u) + 1.7e-3 u o_max T v, and
//    |d(s (c - ln s))| <= |ds| (|c - ln s| + 1) + s (lg2.approx: 1.65e-7 abs,
//    the inner fmaf: u |c - ln s|), |c - ln s| + 1 <= |c| + 89 (s >= 1e-37);
//  * the fp32 running sum of a 32-entry chunk rounds by <= u E1 per step
//    (<= 32 steps per chunk); its fp64 folds are exact to 1e-16;
//  * E1 = sum s (|c - ln s| + 1) needs no per-entry work: sum s <= sum w =
//    1 - T*_final (telescoping) <= W = 1 - T* + eps_T T*, and
//    sum s |ln s| = H_e - c sum s <= H_e + max(0, -c) W (H_e the entries' part
//    of H), so E1 <= (|c| + 1) W + max(0, H_e + max(0, -c) W);
//  * W0 = sum w (1 - v) is within (eps_T + 75 u) W0 + 1.7e-3 u o_max k, and
//    H0 = W0 (c0 - ln W0) moves by at most |dW0| max |c0 - ln W - 1| over
//    [W0 - dW0, W0 + dW0] (or 2 (W0 + dW0)(|c0| + 1 + |ln(W0 + dW0)|) if that
//    interval reaches 0).
// The 1.01 factor covers evaluating the bound from computed (fp32) quantities.
__device__ __forceinline__ double score_bound_px(const UaBlendArgs& a, double He, double W0, double Te,
                                                 int k, float Se) {
  const double u = 5.9604644775390625e-8;
  const double eps_t = 0.5 * (double)cert_window_of(a, (float)k, Se);
  const double W = fmin(1.0, 1.0 - Te + eps_t * Te);
  const double cneg = fmax(0.0, -a.c_ent);
  const double e1 = (fabs(a.c_ent) + 1.0) * W + fmax(0.0, 1.001 * He + cneg * W);
  // (+ 1e-36 per entry: terms of s below fp32's normal range, flushed to zero)
  double b = (eps_t + 76.0 * u + 1.65e-7) * e1 + (a.bound_tail + 1e-36) * (double)k;
  const double dw = (eps_t + 75.0 * u) * W0 + a.w0_tail * (double)k;
  if (W0 > dw) {
    const double lm = fmax(fabs(log(W0 - dw)), fabs(log(W0 + dw)));
    b += dw * (a.c0_abs + 1.0 + lm);
  } else {
    const double wt = W0 + dw;
    b += wt > 0.0 ? 2.0 * wt * (a.c0_abs + 1.0 + fabs(log(wt))) : 0.0;
  }
  return 1.01 * b + 1e-12 * (fabs(He) + W0);
}

// Distance of a track's termination tests from the cutoff, relative.
__device__ __forceinline__ float stop_margin(bool done, float T, float Tprev, float cutoff) {
  const float d = done ? fminf(cutoff - T, Tprev - cutoff) : T - cutoff;
  return d / cutoff;
}

// Two list entries a, b (in list order) composited into one pixel, straight-line:
// an entry the pixel does not cover, or one past its termination, gets alpha = 0.
template <int LC, bool RGB, bool ENT, bool EXTRA>
__device__ __forceinline__ void blend_pair(FPix<LC>& P, const FGeo& ea, const FGeo& eb,
                                           const float4& ua, const float4& ub, bool ca, bool cb,
                                           double cxp, double cyp, float3 cola, float3 colb,
                                           float amax, float cutoff) {
  // q in fp64 (splat_alpha, raster.hpp:101-108), then exp on the SFU
  const double dxa = cxp - ea.mx, dya = cyp - ea.my;
  const double dxb = cxp - eb.mx, dyb = cyp - eb.my;
  const double qa = fma(dxa, fma(ea.cb2, dya, ea.ca * dxa), ea.cc * dya * dya);
  const double qb = fma(dxb, fma(eb.cb2, dyb, eb.ca * dxb), eb.cc * dyb * dyb);
  const float ala = fminf(ea.o * ex2_approx((float)qa * kNegHalfLog2e), amax);
  const float alb = fminf(eb.o * ex2_approx((float)qb * kNegHalfLog2e), amax);
  if (RGB) {
    const bool ra = ca && !P.rd;
    const float aa = ra ? ala : 0.f;
    const float wa = aa * P.T;
    P.r0 = fmaf(wa, cola.x, P.r0);
    P.r1 = fmaf(wa, cola.y, P.r1);
    P.r2 = fmaf(wa, cola.z, P.r2);
    if (EXTRA) P.dp = fmaf(wa, ea.depth, P.dp);
    const float fa = 1.f - aa;
    P.S = fmaf(aa, rcp_approx(fa), P.S);
    const float Ta = fmaf(-P.T, aa, P.T);  // T (1 - a), one rounding
    const bool sa = ra && Ta < cutoff;
    P.Tp = sa ? P.T : P.Tp;
    P.T = Ta;
    const bool rb = cb && !(P.rd || sa);
    const float ab = rb ? alb : 0.f;
    const float wb = ab * P.T;
    P.r0 = fmaf(wb, colb.x, P.r0);
    P.r1 = fmaf(wb, colb.y, P.r1);
    P.r2 = fmaf(wb, colb.z, P.r2);
    if (EXTRA) P.dp = fmaf(wb, eb.depth, P.dp);
    const float fb = 1.f - ab;
    P.S = fmaf(ab, rcp_approx(fb), P.S);
    const float Tb = fmaf(-P.T, ab, P.T);
    const bool sb = rb && Tb < cutoff;
    P.Tp = sb ? P.T : P.Tp;
    P.T = Tb;
    P.rd = P.rd || sa || sb;
    P.n_rgb += (int)ra + (int)rb;
  }
  if (ENT) {
    // compensated_alpha (uncertainty.hpp:55-59) and the entropy step (:198-222);
    // ua = (A, B, v, hl + C_H)
    const bool oa = ca && !P.edn;
    // A, B >= 0 (A = v + beta (1 - v), B = o0 (1 - beta)(1 - v)): no lower clamp needed
    const float xa = fminf(fmaf(ua.x, ala, ua.y), amax);
    const float xb = fminf(fmaf(ub.x, alb, ub.y), amax);
    const float asa = oa ? xa : 0.f;
    const float wa = asa * P.Te;
    const float sa = wa * ua.z;
    P.w0 = fmaf(wa, 1.f - ua.z, P.w0);
    if (EXTRA) P.ed = fmaf(wa, ea.depth, P.ed);
    const float fa = 1.f - asa;
    P.Se = fmaf(asa, rcp_approx(fa), P.Se);
    const float Ta = fmaf(-P.Te, asa, P.Te);
    const bool ta = oa && Ta < cutoff;
    P.Tep = ta ? P.Te : P.Tep;
    P.Te = Ta;
    const bool ob = cb && !(P.edn || ta);
    const float asb = ob ? xb : 0.f;
    const float wb = asb * P.Te;
    const float sb = wb * ub.z;
    P.w0 = fmaf(wb, 1.f - ub.z, P.w0);
    if (EXTRA) P.ed = fmaf(wb, eb.depth, P.ed);
    const float fb = 1.f - asb;
    P.Se = fmaf(asb, rcp_approx(fb), P.Se);
    const float Tb = fmaf(-P.Te, asb, P.Te);
    const bool tb = ob && Tb < cutoff;
    P.Tep = tb ? P.Te : P.Tep;
    P.Te = Tb;
    P.edn = P.edn || ta || tb;
    P.n_ent += (int)oa + (int)ob;
    // H += s (-ln s + 1/2 ln|Qc| + C_H); s == 0 adds exactly 0
    const float la = lg2_approx(fmaxf(sa, 1e-37f));
    const float lb = lg2_approx(fmaxf(sb, 1e-37f));
    const float tta = fmaf(-la, kLn2f, ua.w), ttb = fmaf(-lb, kLn2f, ub.w);
    P.h = fmaf(sa, tta, P.h);
    P.h = fmaf(sb, ttb, P.h);
  }
}

// Word index of the fp16 hi pair w (k = 2w, 2w+1) of entry e, channel ch in a
// staged colour area, and the offset of the matching lo pair.
struct ColWordsStaged {  // fstage_batch: [e][hi: ch][8] [lo: ch][8], 52 words per entry
  static constexpr int kLo = 24;
  __device__ __forceinline__ int operator()(int e, int ch, int w) const {
    return e * kColWords + ch * 8 + w;
  }
};

// One staged batch of n list entries composited into the warp's 32 pixels: warp
// pre-filter per 32-entry chunk, hit entries in groups of 8 (their colours on the
// tensor cores when MMA), two entries at a time through blend_pair.
template <int LC, bool RGB, bool ENT, bool EXTRA, bool MMA, class CW>
__device__ __forceinline__ void blend_batch(FPix<LC>& P, int n, const FGeo* s_geo, const int4* s_rect,
                                            const float4* s_ua, const void* s_col, CW colword,
                                            float* tr, const uint32_t (&aH)[2][4],
                                            const uint32_t (&aL)[2][4], const float2* bp, int lane,
                                            int bx0, int by0, int bx1, int by1, int px, int py,
                                            double cxp,
                                            double cyp, float amax, float cutoff) {
  constexpr int CS = Col<LC>::STRIDE;
  const int gq = lane >> 2, tig = lane & 3;  // mma fragment coordinates
    for (int j0 = 0; j0 < n; j0 += 32) {
      if (__all_sync(0xffffffffu, P.rd && P.edn)) break;  // every pixel of the warp finished
      bool hit = false;
      if (j0 + lane < n) {
        const int4 r = s_rect[j0 + lane];
        hit = r.x <= bx1 && r.x + r.y >= bx0 && r.z <= by1 && r.z + r.w >= by0;
      }
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      if (hits == 0u) continue;
      while (hits != 0u) {
        // the next (up to) 8 hit entries, in list order
        int je[8];
        int ng = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          je[q] = hits != 0u ? j0 + __ffs(hits) - 1 : -1;
          ng += hits != 0u ? 1 : 0;
          hits &= hits - 1u;
        }
        if (RGB && MMA && __any_sync(0xffffffffu, !P.rd)) {
          int my_e = -1;  // B fragment column gq = entry gq of the group
#pragma unroll
          for (int q = 0; q < 8; ++q) my_e = gq == q ? je[q] : my_e;
          uint32_t bh[3][2], bl[3][2];
          const uint32_t* cw = reinterpret_cast<const uint32_t*>(s_col);
          const int e = max(my_e, 0);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int w0 = colword(e, ch, tig), w1 = colword(e, ch, tig + 4);
            bh[ch][0] = my_e >= 0 ? cw[w0] : 0u;
            bh[ch][1] = my_e >= 0 ? cw[w1] : 0u;
            bl[ch][0] = my_e >= 0 ? cw[w0 + CW::kLo] : 0u;
            bl[ch][1] = my_e >= 0 ? cw[w1 + CW::kLo] : 0u;
          }
#pragma unroll
          for (int m = 0; m < 2; ++m) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              float d[4] = {0.f, 0.f, 0.f, 0.f};
              hmma16816(d, aH[m], bh[ch][0], bh[ch][1]);
              hmma16816(d, aH[m], bl[ch][0], bl[ch][1]);
              hmma16816(d, aL[m], bh[ch][0], bh[ch][1]);
              // C fragment: (row gq | gq+8, cols 2 tig, 2 tig + 1) -> [pixel][channel][entry]
              const int r0 = 16 * m + gq, r1 = r0 + 8;
              *reinterpret_cast<float2*>(tr + tr_idx(r0, ch * 8 + 2 * tig)) = make_float2(d[0], d[1]);
              *reinterpret_cast<float2*>(tr + tr_idx(r1, ch * 8 + 2 * tig)) = make_float2(d[2], d[3]);
            }
          }
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          if (q < ng) {
            const int ja = je[q];
            const bool has_b = q + 1 < ng;
            const int jb = has_b ? je[q + 1] : ja;
            const bool ca = in_rect4(s_rect[ja], px, py);
            const bool cb = has_b && in_rect4(s_rect[jb], px, py);
            float3 cola = make_float3(0.f, 0.f, 0.f), colb = cola;
            if (RGB && MMA) {  // entries q, q+1 of the group, own pixel row
              const float2 r = *reinterpret_cast<const float2*>(tr + tr_idx(lane, q));
              const float2 g = *reinterpret_cast<const float2*>(tr + tr_idx(lane, 8 + q));
              const float2 b = *reinterpret_cast<const float2*>(tr + tr_idx(lane, 16 + q));
              cola = make_float3(__saturatef(r.x), __saturatef(g.x), __saturatef(b.x));
              colb = make_float3(__saturatef(r.y), __saturatef(g.y), __saturatef(b.y));
            }
            if (RGB && !MMA) {
              const float* sc = reinterpret_cast<const float*>(s_col);
              sh_color<LC>(reinterpret_cast<const float2*>(sc + ja * CS), bp, cola.x, cola.y, cola.z);
              sh_color<LC>(reinterpret_cast<const float2*>(sc + jb * CS), bp, colb.x, colb.y, colb.z);
            }
            const float4 ua = ENT ? s_ua[ja] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 ub = ENT ? s_ua[jb] : make_float4(0.f, 0.f, 0.f, 0.f);
            blend_pair<LC, RGB, ENT, EXTRA>(P, s_geo[ja], s_geo[jb], ua, ub, ca, cb, cxp, cyp, cola,
                                            colb, amax, cutoff);
          }
        }
        if (RGB && MMA) __syncwarp();  // the next group overwrites the colour block
      }
      fold<LC, EXTRA>(P);
    }
}

// ---------------------------------------------------------------------------
// K7f: 16x16 tiles, 256 threads, one pixel each (warp = 8x4 patch, lane = GEMM
// row), shared-memory batches of the tile list, warp pre-filter (one lane per
// entry against the warp's patch), hit entries in groups of 8 (colours for the
// group on the tensor cores when MMA), composited two at a time.
template <int LC, bool RGB, bool ENT, bool EXTRA, bool MMA, int B>
__global__ void __launch_bounds__(256, kFastMinBlocks) ua_blend_fast_kernel(UaBlendArgs a) {
  using St = FStage<LC, RGB, ENT, MMA>;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  FGeo* s_geo = reinterpret_cast<FGeo*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + B * sizeof(FGeo));
  float4* s_ua = reinterpret_cast<float4*>(s_dyn + B * (sizeof(FGeo) + sizeof(int4)));
  unsigned char* s_col = s_dyn + B * (sizeof(FGeo) + sizeof(int4) + (ENT ? sizeof(float4) : 0));
  float* s_tr = reinterpret_cast<float*>(s_col + (RGB ? B * St::col_bytes() : 0));

  const float amax = (float)a.amax, cutoff = (float)a.cutoff;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tig = lane & 3;  // mma fragment coordinates
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;

  // warp -> an 8x4 pixel patch of the tile (tried: 16x2 strips 9% slower, rows w
  // and w+8 39% slower -- the pre-filter box matters more than warp balance)
  const int bx0 = tx * 16 + (warp & 1) * 8, by0 = ty * 16 + (warp >> 1) * 4;
  const int bx1 = bx0 + 7, by1 = by0 + 3;
  const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
  const bool inside = px < c.width && py < c.height;
  const double cxp = px + 0.5, cyp = py + 0.5;
  FPix<LC> P;
  float2 bp[Col<LC>::NP];           // FFMA colour: SH basis at the pixel ray
  uint32_t aH[2][4], aL[2][4];      // MMA colour: A fragments (rows = lanes), fp16 hi / lo
  float* tr = s_tr + warp * 32 * kTrStride;
  if (RGB && !MMA) pixel_basis<LC>(c, px, py, bp);
  if (RGB && MMA) {
    constexpr int NB = Col<LC>::NB;
    double bd[Col<LC>::NBP];
    pixel_basis_d<LC>(c, px, py, bd);
    uint32_t* wb = reinterpret_cast<uint32_t*>(tr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float x0 = 2 * i < NB ? (float)bd[2 * i] : 0.f;
      const float x1 = 2 * i + 1 < NB ? (float)bd[2 * i + 1] : 0.f;
      uint32_t h, l;
      split_half2(x0, x1, h, l);
      wb[lane * 17 + i] = h;
      wb[lane * 17 + 8 + i] = l;
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int r0 = 16 * m + gq, r1 = r0 + 8;
      aH[m][0] = wb[r0 * 17 + tig];
      aH[m][1] = wb[r1 * 17 + tig];
      aH[m][2] = wb[r0 * 17 + tig + 4];
      aH[m][3] = wb[r1 * 17 + tig + 4];
      aL[m][0] = wb[r0 * 17 + 8 + tig];
      aL[m][1] = wb[r1 * 17 + 8 + tig];
      aL[m][2] = wb[r0 * 17 + 8 + tig + 4];
      aL[m][3] = wb[r1 * 17 + 8 + tig + 4];
    }
    __syncwarp();
  }
  P.T = P.Te = 1.f;
  P.Tp = P.Tep = 1.f;
  P.r0 = P.r1 = P.r2 = P.dp = P.h = P.w0 = P.ed = 0.f;
  P.R0 = P.R1 = P.R2 = P.DP = P.H = P.W0 = P.ED = 0.0;
  P.n_rgb = P.n_ent = 0;
  P.S = P.Se = 0.f;
  P.rd = !(RGB && inside);
  P.edn = !(ENT && inside);

  for (uint32_t base = rg.x; base < rg.y; base += B) {
    const bool live = !(P.rd && P.edn);
    if (__syncthreads_count(live) == 0) break;
    const int n = min((uint32_t)B, rg.y - base);
    fstage_batch<LC, RGB, ENT, MMA>(a, geo, uar, base, n, s_geo, s_rect, s_ua, s_col);
    __syncthreads();
    if (__all_sync(0xffffffffu, !live)) continue;
    blend_batch<LC, RGB, ENT, EXTRA, MMA>(P, n, s_geo, s_rect, s_ua, s_col, ColWordsStaged{}, tr, aH, aL,
                                          bp, lane, bx0, by0, bx1, by1, px, py, cxp, cyp, amax,
                                          cutoff);
  }

  // certification of the stop decisions
  bool flag = false;
  if (inside) {
    if (RGB)
      flag |= stop_margin(P.rd, P.T, P.Tp, cutoff) <=
              cert_window_of(a, (float)P.n_rgb, P.S);
    if (ENT)
      flag |= stop_margin(P.edn, P.Te, P.Tep, cutoff) <=
              cert_window_of(a, (float)P.n_ent, P.Se);
  }
  const int64_t pix = c.pix_base + (int64_t)py * c.width + px;
  const unsigned fm = __ballot_sync(0xffffffffu, flag);
  if (fm != 0u) {
    const int leader = __ffs(fm) - 1;
    uint32_t slot = 0;
    if (lane == leader) slot = atomicAdd(a.flag_count, (uint32_t)__popc(fm));
    slot = __shfl_sync(0xffffffffu, slot, leader);
    if (flag) a.flag_list[slot + __popc(fm & ((1u << lane) - 1u))] = (uint32_t)pix;
  }
  if (!inside) return;
  if (RGB) {
    if (a.rgb) {
      a.rgb[pix * 3 + 0] = P.R0;
      a.rgb[pix * 3 + 1] = P.R1;
      a.rgb[pix * 3 + 2] = P.R2;
    }
    if (EXTRA && a.depth) a.depth[pix] = P.DP;
    if (a.trans) a.trans[pix] = (double)P.T;
    if (EXTRA && a.rgb_contrib) a.rgb_contrib[pix] = P.n_rgb;
  }
  if (ENT) {
    double H = P.H;
    if (P.W0 > 0.0) H += P.W0 * (-log(P.W0) + a.hl_q0 + kGaussEntropy);  // :224-225
    if (a.score_bound) a.score_bound[pix] = score_bound_px(a, P.H, P.W0, (double)P.Te, P.n_ent, P.Se);
    if (a.entropy) a.entropy[pix] = H;
    if (a.w0) a.w0[pix] = P.W0;
    if (EXTRA && a.edepth) a.edepth[pix] = P.ED;
    if (EXTRA && a.ent_contrib) a.ent_contrib[pix] = P.n_ent;
  }
}

// ---------------------------------------------------------------------------
// K7 exact (fp64 blend) with the tensor-core colour: the fp64 arithmetic of
// ua_blend_ilp_kernel (kernels_ua.cu; the ex_* steps of ua_common.cuh) on K7f's
// staging and colour machinery -- half the CTA stages the fp64 records, the
// other half cp.asyncs the pre-split colour records; per group of 8 hit entries
// the warp's 32 x 24 colour block comes from 18 mma.sync (split fp16, fp32
// accumulate) instead of 8 x (12 LDS.128 + 24 FFMA2) per lane. Only the SH
// colour dot product is affected (split-fp16 operands, ~2^-21 relative, as in
// the certified path); alpha, both transmittances, the stop tests and every
// accumulation stay fp64. GAVIS_UA_COLOR=ffma selects the packed-FFMA kernel.

template <int LC, bool ENT>
__device__ __forceinline__ void estage_batch(const UaBlendArgs& a, const GeoRec* geo, const UaRec* uar,
                                             uint32_t base, int n, ExGeo* s_geo, int4* s_rect,
                                             ExUa* s_ua, uint32_t* s_col) {
  constexpr int kHalf = 128;
  const int t = threadIdx.x;
  if (t >= kHalf) {
    uint4* dst = reinterpret_cast<uint4*>(s_col);
    for (int j = t - kHalf; j < n; j += kHalf) {
      const uint4* src = a.scene.colors_split + (int64_t)a.vals[base + j] * (kColWords / 4);
#pragma unroll
      for (int w = 0; w < kColWords / 4; ++w) cp_async16(dst + j * (kColWords / 4) + w, src + w);
    }
    cp_async_wait_all();
    return;
  }
  for (int j = t; j < n; j += kHalf) {
    const uint32_t g = a.vals[base + j];
    const GeoRec r = geo[g];
    s_geo[j] = ex_geo(r);
    s_rect[j] = cover_rect4(r.cov_x, r.cov_y);
    if (ENT) s_ua[j] = ex_ua(uar[g]);
  }
}

// Two list entries composited in fp64 (the pair step of ua_blend_ilp_kernel).
// A track's update is masked for lanes whose pixel the entry does not cover (or
// whose track is done) by zeroing its alpha with a select (alpha = 0 adds +0 and
// multiplies T by exactly 1). GAVIS_PRED_TRACKS=1 guards the updates with `if`s
// instead -- bit-identical, two FSELs fewer per track and entry, but the compiler
// turns the entropy blocks into divergent branches: 1404 vs 1518 views/s.
#ifndef GAVIS_PRED_TRACKS
#define GAVIS_PRED_TRACKS 0
#endif
template <int LC, bool ENT, bool EXTRA, bool LO, class Rec>
__device__ __forceinline__ void exact_pair(Pixel<LC>& P, const Rec& ea, const Rec& eb, const ExUa& ua,
                                           const ExUa& ub, bool ca, bool cb, double cxp, double cyp,
                                           float3 cola, float3 colb, double amax, double cutoff) {
  const double ala = ex_alpha(ea, ex_negq(ea, cxp, cyp), amax);
  const double alb = ex_alpha(eb, ex_negq(eb, cxp, cyp), amax);
  const bool ra = ca && !P.rgb_done;
#if GAVIS_PRED_TRACKS >= 1
  if (ra) ex_rgb<LC, EXTRA, LO>(P, ala, ea.depth, cola.x, cola.y, cola.z);
#else
  ex_rgb<LC, EXTRA, LO>(P, ra ? ala : 0.0, ea.depth, cola.x, cola.y, cola.z);
#endif
  const bool rd = P.rgb_done || (ra && P.T < cutoff);
  const bool rb = cb && !rd;
#if GAVIS_PRED_TRACKS >= 1
  if (rb) ex_rgb<LC, EXTRA, LO>(P, alb, eb.depth, colb.x, colb.y, colb.z);
#else
  ex_rgb<LC, EXTRA, LO>(P, rb ? alb : 0.0, eb.depth, colb.x, colb.y, colb.z);
#endif
  if (EXTRA) P.n_rgb += (int)ra + (int)rb;
  P.rgb_done = rd || (rb && P.T < cutoff);
  if (ENT) {
    const double xa = ex_astar<LO>(ua, ala, amax), xb = ex_astar<LO>(ub, alb, amax);
    const bool ea_on = ca && !P.ent_done;
#if GAVIS_PRED_TRACKS == 1
    double sa = 0.0;
    if (ea_on) sa = ex_ent<LC, EXTRA>(P, xa, ua, ea.depth);
#else
    const double sa = ex_ent<LC, EXTRA>(P, ea_on ? xa : 0.0, ua, ea.depth);
#endif
    const bool ed = P.ent_done || (ea_on && P.Te < cutoff);
    const bool eb_on = cb && !ed;
#if GAVIS_PRED_TRACKS == 1
    double sb = 0.0;
    if (eb_on) sb = ex_ent<LC, EXTRA>(P, xb, ub, eb.depth);
#else
    const double sb = ex_ent<LC, EXTRA>(P, eb_on ? xb : 0.0, ub, eb.depth);
#endif
    if (LO) {  // s may be negative (given visibility outside [0, 1]): s > 0 only
      const double la = log_blend(sa > 0.0 ? sa : 1.0);
      const double lb = log_blend(sb > 0.0 ? sb : 1.0);
      if (sa > 0.0) P.H = fma(sa, ua.hlc - la, P.H);
      if (sb > 0.0) P.H = fma(sb, ub.hlc - lb, P.H);
    } else {  // s >= 0; s == 0 adds exactly +0 (log_blend(0) is finite)
      P.H = fma(sa, ua.hlc - log_blend(sa), P.H);
      P.H = fma(sb, ub.hlc - log_blend(sb), P.H);
    }
    if (EXTRA) P.n_ent += (int)ea_on + (int)eb_on;
    P.ent_done = ed || (eb_on && P.Te < cutoff);
  }
}

#ifndef GAVIS_EXACT_MIN_BLOCKS
#define GAVIS_EXACT_MIN_BLOCKS 4
#define GAVIS_EXACT_BATCH 64
#endif
// 4 CTAs per SM: 64 registers (the same 12-byte spill as at 80) and 64-entry
// batches (53.6 KB of shared memory each): 32 warps per SM instead of 24,
// 1482 vs 1462 views/s at config 3 over 3 CTAs of 128-entry batches
constexpr int kExactMinBlocks = GAVIS_EXACT_MIN_BLOCKS;
constexpr int kExactBatch = GAVIS_EXACT_BATCH;

template <bool ENT>
struct EStage {
  static constexpr size_t bytes(int batch) {
    return (size_t)batch * (sizeof(ExGeo) + sizeof(int4) + (ENT ? sizeof(ExUa) : 0) +
                            sizeof(uint32_t) * kColWords) +
           8 * 32 * kTrStride * sizeof(float);
  }
};

template <int LC, bool ENT, bool EXTRA, bool LO, int B>
__global__ void __launch_bounds__(256, kExactMinBlocks) ua_blend_exact_mma_kernel(UaBlendArgs a) {
  extern __shared__ __align__(16) unsigned char s_dyn[];
  ExGeo* s_geo = reinterpret_cast<ExGeo*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + B * sizeof(ExGeo));
  ExUa* s_ua = reinterpret_cast<ExUa*>(s_dyn + B * (sizeof(ExGeo) + sizeof(int4)));
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_dyn + B * (sizeof(ExGeo) + sizeof(int4) +
                                                             (ENT ? sizeof(ExUa) : 0)));
  float* s_tr = reinterpret_cast<float*>(s_col + B * kColWords);
  load_math_tables();

  const double amax = a.amax, cutoff = a.cutoff;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tig = lane & 3;  // mma fragment coordinates
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;

  const int bx0 = tx * 16 + (warp & 1) * 8, by0 = ty * 16 + (warp >> 1) * 4;
  const int bx1 = bx0 + 7, by1 = by0 + 3;
  const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
  const bool inside = px < c.width && py < c.height;
  const double cxp = px + 0.5, cyp = py + 0.5;
  float* tr = s_tr + warp * 32 * kTrStride;
  uint32_t aH[2][4], aL[2][4];  // A fragments of the pixel SH basis (rows = lanes), fp16 hi / lo
  {
    constexpr int NB = Col<LC>::NB;
    double bd[Col<LC>::NBP];
    pixel_basis_d<LC>(c, px, py, bd);
    uint32_t* wb = reinterpret_cast<uint32_t*>(tr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float x0 = 2 * i < NB ? (float)bd[2 * i] : 0.f;
      const float x1 = 2 * i + 1 < NB ? (float)bd[2 * i + 1] : 0.f;
      uint32_t h, l;
      split_half2(x0, x1, h, l);
      wb[lane * 17 + i] = h;
      wb[lane * 17 + 8 + i] = l;
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int r0 = 16 * m + gq, r1 = r0 + 8;
      aH[m][0] = wb[r0 * 17 + tig];
      aH[m][1] = wb[r1 * 17 + tig];
      aH[m][2] = wb[r0 * 17 + tig + 4];
      aH[m][3] = wb[r1 * 17 + tig + 4];
      aL[m][0] = wb[r0 * 17 + 8 + tig];
      aL[m][1] = wb[r1 * 17 + 8 + tig];
      aL[m][2] = wb[r0 * 17 + 8 + tig + 4];
      aL[m][3] = wb[r1 * 17 + 8 + tig + 4];
    }
    __syncwarp();
  }
  Pixel<LC> P;
  P.T = P.Te = 1.0;
  P.rgb0 = P.rgb1 = P.rgb2 = P.dep = 0.0;
  P.H = P.w0 = P.edep = 0.0;
  P.rgb_done = !inside;
  P.ent_done = !(ENT && inside);
  P.n_rgb = P.n_ent = 0;
  const ColWordsStaged colword;

  for (uint32_t base = rg.x; base < rg.y; base += B) {
    const bool live = !(P.rgb_done && P.ent_done);
    if (__syncthreads_count(live) == 0) break;
    const int n = min((uint32_t)B, rg.y - base);
    estage_batch<LC, ENT>(a, geo, uar, base, n, s_geo, s_rect, s_ua, s_col);
    __syncthreads();
    if (__all_sync(0xffffffffu, !live)) continue;
    for (int j0 = 0; j0 < n; j0 += 32) {
      if (__all_sync(0xffffffffu, P.rgb_done && P.ent_done)) break;
      bool hit = false;
      if (j0 + lane < n) {
        const int4 r = s_rect[j0 + lane];
        hit = r.x <= bx1 && r.x + r.y >= bx0 && r.z <= by1 && r.z + r.w >= by0;
      }
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      while (hits != 0u) {
        int je[8];
        int ng = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          je[q] = hits != 0u ? j0 + __ffs(hits) - 1 : -1;
          ng += hits != 0u ? 1 : 0;
          hits &= hits - 1u;
        }
        if (__any_sync(0xffffffffu, !P.rgb_done)) {
          int my_e = -1;  // B fragment column gq = entry gq of the group
#pragma unroll
          for (int q = 0; q < 8; ++q) my_e = gq == q ? je[q] : my_e;
          uint32_t bh[3][2], bl[3][2];
          const int e = max(my_e, 0);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int w0 = colword(e, ch, tig), w1 = colword(e, ch, tig + 4);
            bh[ch][0] = my_e >= 0 ? s_col[w0] : 0u;
            bh[ch][1] = my_e >= 0 ? s_col[w1] : 0u;
            bl[ch][0] = my_e >= 0 ? s_col[w0 + ColWordsStaged::kLo] : 0u;
            bl[ch][1] = my_e >= 0 ? s_col[w1 + ColWordsStaged::kLo] : 0u;
          }
#pragma unroll
          for (int m = 0; m < 2; ++m) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              float d[4] = {0.f, 0.f, 0.f, 0.f};
              hmma16816(d, aH[m], bh[ch][0], bh[ch][1]);
              hmma16816(d, aH[m], bl[ch][0], bl[ch][1]);
              hmma16816(d, aL[m], bh[ch][0], bh[ch][1]);
              const int r0 = 16 * m + gq, r1 = r0 + 8;
              *reinterpret_cast<float2*>(tr + tr_idx(r0, ch * 8 + 2 * tig)) = make_float2(d[0], d[1]);
              *reinterpret_cast<float2*>(tr + tr_idx(r1, ch * 8 + 2 * tig)) = make_float2(d[2], d[3]);
            }
          }
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          if (q < ng) {
            const int ja = je[q];
            const bool has_b = q + 1 < ng;
            const int jb = has_b ? je[q + 1] : ja;
            const bool ca = in_rect4(s_rect[ja], px, py);
            const bool cb = has_b && in_rect4(s_rect[jb], px, py);
            const float2 r = *reinterpret_cast<const float2*>(tr + tr_idx(lane, q));
            const float2 g = *reinterpret_cast<const float2*>(tr + tr_idx(lane, 8 + q));
            const float2 b = *reinterpret_cast<const float2*>(tr + tr_idx(lane, 16 + q));
            const float3 cola = make_float3(__saturatef(r.x), __saturatef(g.x), __saturatef(b.x));
            const float3 colb = make_float3(__saturatef(r.y), __saturatef(g.y), __saturatef(b.y));
            exact_pair<LC, ENT, EXTRA, LO>(P, s_geo[ja], s_geo[jb], s_ua[ENT ? ja : 0], s_ua[ENT ? jb : 0], ca,
                                           cb, cxp, cyp, cola, colb, amax, cutoff);
          }
        }
        __syncwarp();  // the next group overwrites the colour block
      }
    }
  }
  pixel_finish<LC, true, ENT, EXTRA>(P, a, c, px, py, inside);
}

// ---------------------------------------------------------------------------
// K7 exact, TMA ring (opt-in, GAVIS_UA_RING=1; measured slower): the same fp64
// blend and tensor-core colour as ua_blend_exact_mma_kernel, but the tile list
// streams through a ring of kRing slots of 32 entries filled by bulk copies
// (cp.async.bulk, completion on an mbarrier per slot) instead of staged batches
// between two CTA barriers. The 8 warps are decoupled: a warp waits only for
// the slot it reads to land, never for the other warps (the block barriers and
// their per-batch wait for the slowest warp were ~19% of the stall samples).
// A slot is refilled by the LAST warp to release it (a shared-memory arrival
// counter), so no producer warp and no extra registers: the 32 lanes of that
// warp read the next 32 particle ids and issue the record copies (GeoRec 64 B,
// UaRec 48 B, split colour record 208 B per entry) directly from the K1/scene
// arrays. The per-slot tag (batch held, or STOP) orders the refill decision
// before any warp waits on the slot: once every warp's pixels are done the ring
// stops refilling and each warp leaves at the first STOP, with no copy in
// flight (every issued slot was waited on before its successor was decided).
#ifndef GAVIS_RING_SLOTS
#define GAVIS_RING_SLOTS 4
#define GAVIS_RING_MIN_BLOCKS 3
#endif
constexpr int kRing = GAVIS_RING_SLOTS;
constexpr int kRingMinBlocks = GAVIS_RING_MIN_BLOCKS;
constexpr int kRingEntries = 32;
constexpr int kRingStop = -1;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Sleep until the phase with `parity` completes: try_wait with a suspend-time
// hint parks the warp in hardware (a bare try_wait returns after a short
// system-dependent time, and re-issuing it from a C++ loop cost as many issue
// slots as the blend itself: 5.6 G extra warp instructions per 16 views).
#ifndef GAVIS_WAIT_HINT_NS
#define GAVIS_WAIT_HINT_NS 2000
#endif
constexpr uint32_t kWaitHintNs = GAVIS_WAIT_HINT_NS;  // ~ one bulk-copy latency
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      " @!p bra WAIT;\n}"
      ::"r"(smem_u32(bar)), "r"(parity), "r"(kWaitHintNs)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <bool ENT>
struct RingLayout {
  static constexpr size_t geo = (size_t)kRing * kRingEntries * sizeof(GeoRec);
  static constexpr size_t ua = ENT ? (size_t)kRing * kRingEntries * sizeof(UaRec) : 0;
  static constexpr size_t col = (size_t)kRing * kRingEntries * kColWords * sizeof(uint32_t);
  static constexpr size_t tr = 8 * 32 * kTrStride * sizeof(float);
  static constexpr size_t bytes = geo + ua + col + tr;
  static constexpr uint32_t entry_bytes =
      (uint32_t)(sizeof(GeoRec) + (ENT ? sizeof(UaRec) : 0) + kColWords * sizeof(uint32_t));
};

// Lane j of the calling warp issues the copies of entry j of list batch `bi`
// into ring slot `slot` (lane 0 first arms the slot's barrier with the bytes).
template <bool ENT>
__device__ __forceinline__ void ring_issue(const UaBlendArgs& a, const GeoRec* geo, const UaRec* uar,
                                           uint2 rg, int bi, int slot, int lane, GeoRec* s_geo, UaRec* s_ua,
                                           uint32_t* s_col, uint64_t* full) {
  const uint32_t base = rg.x + (uint32_t)bi * kRingEntries;
  const int n = (int)min((uint32_t)kRingEntries, rg.y - base);
  if (lane == 0) mbar_arrive_expect_tx(&full[slot], (uint32_t)n * RingLayout<ENT>::entry_bytes);
  __syncwarp();
  if (lane < n) {
    const uint32_t g = a.vals[base + lane];
    const int e = slot * kRingEntries + lane;
    bulk_g2s(s_geo + e, geo + g, sizeof(GeoRec), &full[slot]);
    if (ENT) bulk_g2s(s_ua + e, uar + g, sizeof(UaRec), &full[slot]);
    bulk_g2s(s_col + (size_t)e * kColWords, a.scene.colors_split + (int64_t)g * (kColWords / 4),
             kColWords * sizeof(uint32_t), &full[slot]);
  }
}

template <int LC, bool ENT, bool EXTRA, bool LO>
__global__ void __launch_bounds__(256, kRingMinBlocks) ua_blend_exact_tma_kernel(UaBlendArgs a) {
  using L = RingLayout<ENT>;
  extern __shared__ __align__(128) unsigned char s_dyn[];
  GeoRec* s_geo = reinterpret_cast<GeoRec*>(s_dyn);
  UaRec* s_ua = reinterpret_cast<UaRec*>(s_dyn + L::geo);
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_dyn + L::geo + L::ua);
  float* s_tr = reinterpret_cast<float*>(s_dyn + L::geo + L::ua + L::col);
  __shared__ __align__(8) uint64_t full[kRing];
  __shared__ int s_tag[kRing];
  __shared__ int s_rel[kRing];
  __shared__ int s_ndone;
  load_math_tables();

  const double amax = a.amax, cutoff = a.cutoff;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int nbatch = (int)((rg.y - rg.x + kRingEntries - 1) / kRingEntries);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tig = lane & 3;
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;

  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) {
      mbar_init(&full[s], 1);
      s_tag[s] = s < nbatch ? s : kRingStop;
      s_rel[s] = 0;
    }
    s_ndone = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int s = 0; s < kRing && s < nbatch; ++s) ring_issue<ENT>(a, geo, uar, rg, s, s, lane, s_geo, s_ua, s_col, full);

  const int bx0 = tx * 16 + (warp & 1) * 8, by0 = ty * 16 + (warp >> 1) * 4;
  const int bx1 = bx0 + 7, by1 = by0 + 3;
  const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
  const bool inside = px < c.width && py < c.height;
  const double cxp = px + 0.5, cyp = py + 0.5;
  float* tr = s_tr + warp * 32 * kTrStride;
  uint32_t aH[2][4], aL[2][4];
  {
    constexpr int NB = Col<LC>::NB;
    double bd[Col<LC>::NBP];
    pixel_basis_d<LC>(c, px, py, bd);
    uint32_t* wb = reinterpret_cast<uint32_t*>(tr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float x0 = 2 * i < NB ? (float)bd[2 * i] : 0.f;
      const float x1 = 2 * i + 1 < NB ? (float)bd[2 * i + 1] : 0.f;
      uint32_t h, l;
      split_half2(x0, x1, h, l);
      wb[lane * 17 + i] = h;
      wb[lane * 17 + 8 + i] = l;
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const int r0 = 16 * m + gq, r1 = r0 + 8;
      aH[m][0] = wb[r0 * 17 + tig];
      aH[m][1] = wb[r1 * 17 + tig];
      aH[m][2] = wb[r0 * 17 + tig + 4];
      aH[m][3] = wb[r1 * 17 + tig + 4];
      aL[m][0] = wb[r0 * 17 + 8 + tig];
      aL[m][1] = wb[r1 * 17 + 8 + tig];
      aL[m][2] = wb[r0 * 17 + 8 + tig + 4];
      aL[m][3] = wb[r1 * 17 + 8 + tig + 4];
    }
    __syncwarp();
  }
  Pixel<LC> P;
  P.T = P.Te = 1.0;
  P.rgb0 = P.rgb1 = P.rgb2 = P.dep = 0.0;
  P.H = P.w0 = P.edep = 0.0;
  P.rgb_done = !inside;
  P.ent_done = !(ENT && inside);
  P.n_rgb = P.n_ent = 0;
  const ColWordsStaged colword;
  bool counted = false;  // this warp's pixels are all done and s_ndone knows it

  for (int bi = 0; bi < nbatch; ++bi) {
    const int slot = bi % kRing;
    // The slot's barrier phase for batch bi completes either when its copies land
    // or, once the ring stops, by a plain arrival of the deciding warp; the tag
    // (written before either) says which. The wait sleeps in hardware.
    mbar_wait(&full[slot], (uint32_t)((bi / kRing) & 1));
    if (((volatile int*)s_tag)[slot] == kRingStop) break;
    const bool wdone = __all_sync(0xffffffffu, P.rgb_done && P.ent_done);
    if (!wdone) {
      const int n = (int)min((uint32_t)kRingEntries, rg.y - (rg.x + (uint32_t)bi * kRingEntries));
      const GeoRec* sg = s_geo + slot * kRingEntries;
      const UaRec* su = s_ua + slot * kRingEntries;
      const uint32_t* sc = s_col + (size_t)slot * kRingEntries * kColWords;
      bool hit = false;
      if (lane < n) {
        const int4 r = cover_rect4(sg[lane].cov_x, sg[lane].cov_y);
        hit = r.x <= bx1 && r.x + r.y >= bx0 && r.z <= by1 && r.z + r.w >= by0;
      }
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      while (hits != 0u) {
        int je[8];
        int ng = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          je[q] = hits != 0u ? __ffs(hits) - 1 : -1;
          ng += hits != 0u ? 1 : 0;
          hits &= hits - 1u;
        }
        if (__any_sync(0xffffffffu, !P.rgb_done)) {
          int my_e = -1;
#pragma unroll
          for (int q = 0; q < 8; ++q) my_e = gq == q ? je[q] : my_e;
          uint32_t bh[3][2], bl[3][2];
          const int e = max(my_e, 0);
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int w0 = colword(e, ch, tig), w1 = colword(e, ch, tig + 4);
            bh[ch][0] = my_e >= 0 ? sc[w0] : 0u;
            bh[ch][1] = my_e >= 0 ? sc[w1] : 0u;
            bl[ch][0] = my_e >= 0 ? sc[w0 + ColWordsStaged::kLo] : 0u;
            bl[ch][1] = my_e >= 0 ? sc[w1 + ColWordsStaged::kLo] : 0u;
          }
#pragma unroll
          for (int m = 0; m < 2; ++m) {
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) {
              float d[4] = {0.f, 0.f, 0.f, 0.f};
              hmma16816(d, aH[m], bh[ch][0], bh[ch][1]);
              hmma16816(d, aH[m], bl[ch][0], bl[ch][1]);
              hmma16816(d, aL[m], bh[ch][0], bh[ch][1]);
              const int r0 = 16 * m + gq, r1 = r0 + 8;
              *reinterpret_cast<float2*>(tr + tr_idx(r0, ch * 8 + 2 * tig)) = make_float2(d[0], d[1]);
              *reinterpret_cast<float2*>(tr + tr_idx(r1, ch * 8 + 2 * tig)) = make_float2(d[2], d[3]);
            }
          }
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          if (q < ng) {
            const int ja = je[q];
            const bool has_b = q + 1 < ng;
            const int jb = has_b ? je[q + 1] : ja;
            const GeoRec& ga = sg[ja];
            const GeoRec& gb = sg[jb];
            const bool ca = in_rect4(cover_rect4(ga.cov_x, ga.cov_y), px, py);
            const bool cb = has_b && in_rect4(cover_rect4(gb.cov_x, gb.cov_y), px, py);
            const float2 r = *reinterpret_cast<const float2*>(tr + tr_idx(lane, q));
            const float2 g = *reinterpret_cast<const float2*>(tr + tr_idx(lane, 8 + q));
            const float2 b = *reinterpret_cast<const float2*>(tr + tr_idx(lane, 16 + q));
            const float3 cola = make_float3(__saturatef(r.x), __saturatef(g.x), __saturatef(b.x));
            const float3 colb = make_float3(__saturatef(r.y), __saturatef(g.y), __saturatef(b.y));
            exact_pair<LC, ENT, EXTRA, LO>(P, ga, gb, ENT ? ex_ua(su[ja]) : ExUa{},
                                           ENT ? ex_ua(su[jb]) : ExUa{}, ca, cb, cxp, cyp, cola, colb, amax,
                                           cutoff);
          }
        }
        __syncwarp();
      }
    }
    // release the slot; the last of the 8 warps decides its refill
    if (!counted && __all_sync(0xffffffffu, P.rgb_done && P.ent_done)) {
      counted = true;
      if (lane == 0) atomicAdd(&s_ndone, 1);
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(&s_rel[slot], 1) == 7;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      const int next = bi + kRing;
      const bool stop = next >= nbatch || *((volatile int*)&s_ndone) == 8;
      if (lane == 0) s_rel[slot] = 0;
      if (stop) {
        if (lane == 0) {
          ((volatile int*)s_tag)[slot] = kRingStop;
          __threadfence_block();
          mbar_arrive(&full[slot]);  // completes the phase the other warps wait on
        }
      } else {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // slot reads before the copies' writes
        if (lane == 0) {
          ((volatile int*)s_tag)[slot] = next;
          __threadfence_block();
        }
        __syncwarp();
        ring_issue<ENT>(a, geo, uar, rg, next, slot, lane, s_geo, s_ua, s_col, full);
      }
      __syncwarp();
    }
  }
  pixel_finish<LC, true, ENT, EXTRA>(P, a, c, px, py, inside);
}

template <int LC, bool ENT, bool EXTRA, bool LO>
void launch_exact_tma(const UaBlendArgs& a, cudaStream_t s) {
  const size_t sm = RingLayout<ENT>::bytes;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ua_blend_exact_tma_kernel<LC, ENT, EXTRA, LO>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  ua_blend_exact_tma_kernel<LC, ENT, EXTRA, LO><<<(unsigned)a.total_tiles, 256, sm, s>>>(a);
}

// GAVIS_UA_RING=1 selects the TMA-ring kernel (A/B; the barrier-staged kernel
// is the default: 720 vs 765 ms of blend per 1024 views at config 3)
inline bool exact_ring() {
  static const bool ring = [] {
    const char* e = std::getenv("GAVIS_UA_RING");
    return e && e[0] == '1';
  }();
  return ring;
}

template <int LC, bool ENT, bool EXTRA, bool LO>
void launch_exact_mma(const UaBlendArgs& a, cudaStream_t s) {
  if (exact_ring()) {
    launch_exact_tma<LC, ENT, EXTRA, LO>(a, s);
    return;
  }
  constexpr int B = kExactBatch;
  const size_t sm = EStage<ENT>::bytes(B);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ua_blend_exact_mma_kernel<LC, ENT, EXTRA, LO, B>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  ua_blend_exact_mma_kernel<LC, ENT, EXTRA, LO, B><<<(unsigned)a.total_tiles, 256, sm, s>>>(a);
}

template <int LC, bool EXTRA>
void launch_exact_mma_lc(const UaBlendArgs& a, cudaStream_t s) {
  if (a.do_ent) {
    if (a.vis_outside_unit)
      launch_exact_mma<LC, true, EXTRA, true>(a, s);
    else
      launch_exact_mma<LC, true, EXTRA, false>(a, s);
  } else if (a.vis_outside_unit) {  // negative opacities: the RGB w > 0 guard
    launch_exact_mma<LC, false, EXTRA, true>(a, s);
  } else {
    launch_exact_mma<LC, false, EXTRA, false>(a, s);
  }
}

// ---------------------------------------------------------------------------
// K7r: exact fp64 recomputation of the flagged pixels, one warp per pixel.
// The lanes walk the pixel's tile list 32 entries at a time: each lane loads
// its entry, tests coverage and, if covered, evaluates the entry's fp64 alpha,
// compensated alpha and fp32 SH colour (independent of the transmittance).
// The covered entries are then composited in list order with the exact
// path's operations (rgb_step / ent_step, ua_common.cuh), every lane carrying
// the same pixel state, so the outputs equal the exact kernels' bit for bit.
template <int LC, bool RGB, bool ENT>
__global__ void __launch_bounds__(32) ua_redo_kernel(UaBlendArgs a) {
  load_math_tables();
  __syncthreads();
  constexpr int CS = Col<LC>::STRIDE;
  const uint32_t n = *a.flag_count;
  const double amax = a.amax, cutoff = a.cutoff;
  const int64_t N = a.scene.n;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nwarps) {
    const int64_t pix = a.flag_list[i];
    int v = 0;
    while (v + 1 < a.V && a.cams[v + 1].pix_base <= pix) ++v;
    const DevCam& c = a.cams[v];
    const int64_t local = pix - c.pix_base;
    const int py = (int)(local / c.width), px = (int)(local - (int64_t)py * c.width);
    const int64_t tile = c.tile_base + (int64_t)(py / a.tile_size) * c.tiles_x + px / a.tile_size;
    const uint2 rg = a.ranges[tile];
    const GeoRec* geo = a.geo + (int64_t)v * N;
    const UaRec* uar = a.ua + (int64_t)v * N;
    const double cxp = px + 0.5, cyp = py + 0.5;
    Pixel<LC> P;
    pixel_init<LC, RGB, ENT>(P, c, px, py, true);
    for (uint32_t base = rg.x; base < rg.y; base += 32) {
      if (P.rgb_done && P.ent_done) break;
      const uint32_t j = base + lane;
      bool cov = false;
      double al = 0.0, as = 0.0, dep = 0.0, vv = 0.0, omv = 0.0, hlc = 0.0;
      float c0 = 0.f, c1 = 0.f, c2 = 0.f;
      if (j < rg.y) {
        const uint32_t g = a.vals[j];
        const GeoRec r = geo[g];
        cov = in_rect4(cover_rect4(r.cov_x, r.cov_y), px, py);
        if (cov) {
          // the exact kernels' arithmetic (ua_common.cuh), lane-parallel per entry
          const ExGeo e = ex_geo(r);
          al = ex_alpha(e, ex_negq(e, cxp, cyp), amax);
          dep = e.depth;
          if (RGB)
            sh_color<LC>(reinterpret_cast<const float2*>(a.scene.colors + (int64_t)g * CS), P.bp, c0,
                         c1, c2);
          if (ENT) {
            const ExUa u = ex_ua(uar[g]);
            as = ex_astar<true>(u, al, amax);  // the lower clamp is a no-op when A alpha + B >= 0
            vv = u.v;
            omv = u.omv;
            hlc = u.hlc;
          }
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, cov);
      double my_s = 0.0;  // s of this lane's entry if the entropy track composited it
      unsigned mm = m;
      while (mm != 0u) {
        const int src = __ffs(mm) - 1;
        mm &= mm - 1u;
        const double eal = __shfl_sync(0xffffffffu, al, src);
        const double edep = __shfl_sync(0xffffffffu, dep, src);
        if (RGB && !P.rgb_done) {  // rasterize (raster.hpp:209-221)
          const float e0 = __shfl_sync(0xffffffffu, c0, src);
          const float e1 = __shfl_sync(0xffffffffu, c1, src);
          const float e2 = __shfl_sync(0xffffffffu, c2, src);
          ++P.n_rgb;
          ex_rgb<LC, true>(P, eal, edep, e0, e1, e2);
          if (P.T < cutoff) P.rgb_done = true;
        }
        if (ENT && !P.ent_done) {  // render_entropy_core (uncertainty.hpp:198-222), H deferred
          ExUa u = {};
          u.v = __shfl_sync(0xffffffffu, vv, src);
          u.omv = __shfl_sync(0xffffffffu, omv, src);
          const double eas = __shfl_sync(0xffffffffu, as, src);
          ++P.n_ent;
          const double sv = ex_ent<LC, true>(P, eas, u, edep);
          if (lane == src) my_s = sv;
          if (P.Te < cutoff) P.ent_done = true;
        }
        if (P.rgb_done && P.ent_done) break;
      }
      if (ENT) {
        // H += s (-ln s + 1/2 ln|Qc| + C_H) in list order as fma(s, hlc - ln s, H):
        // the logs in parallel (one per lane), the sum serial
        const double tl = my_s > 0.0 ? hlc - log_blend(my_s) : 0.0;
        mm = m;
        while (mm != 0u) {
          const int src = __ffs(mm) - 1;
          mm &= mm - 1u;
          const double ss = __shfl_sync(0xffffffffu, my_s, src);
          const double tt = __shfl_sync(0xffffffffu, tl, src);
          if (ss > 0.0) P.H = fma(ss, tt, P.H);
        }
      }
    }
    if (lane == 0) pixel_finish<LC, RGB, ENT, true>(P, a, c, px, py, true);
  }
}

// K8: image_entropy (uncertainty.hpp:264-278) per view in two fixed-order
// stages: block (chunk, view) folds its pixels (thread t: t, t + 256, ...), a
// shuffle tree and the 8 warp sums in order; then one warp per view folds the
// chunk partials (lane-contiguous blocks, shuffle tree). Deterministic.
constexpr int kScoreChunks = 64;

__global__ void __launch_bounds__(256) score_image_kernel(const DevCam* cams, const double* entropy,
                                                          const double* edepth, double lambda,
                                                          double* partial) {
  __shared__ double s_red[8];
  const DevCam& c = cams[blockIdx.y];
  const int64_t P = (int64_t)c.width * c.height;
  const int64_t lo = P * blockIdx.x / kScoreChunks, hi = P * (blockIdx.x + 1) / kScoreChunks;
  const double* H = entropy + c.pix_base;
  double sum = 0.0;
  if (lambda > 0.0) {
    const double* d = edepth + c.pix_base;
    for (int64_t i = lo + threadIdx.x; i < hi; i += 256) sum += H[i] - H[i] * exp(-d[i] / lambda);
  } else {
    for (int64_t i = lo + threadIdx.x; i < hi; i += 256) sum += H[i];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += s_red[w];
    partial[(int64_t)blockIdx.y * kScoreChunks + blockIdx.x] = s;
  }
}

__global__ void score_fold_kernel(const double* partial, double* scores) {
  const int v = blockIdx.x, lane = threadIdx.x;
  const double* p = partial + (int64_t)v * kScoreChunks;
  double sum = 0.0;
  for (int i = lane * (kScoreChunks / 32); i < (lane + 1) * (kScoreChunks / 32); ++i) sum += p[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if (lane == 0) scores[v] = sum;
}

// batch of 128 list entries (tried 96: +2%, 160: +3%; 192 leaves 2 CTAs per SM)
template <int LC, bool RGB, bool ENT, bool EXTRA, bool MMA, int B>
void launch_fast_kernel_b(const UaBlendArgs& a, cudaStream_t s) {
  using St = FStage<LC, RGB, ENT, MMA>;
  const size_t sm = St::bytes(B);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ua_blend_fast_kernel<LC, RGB, ENT, EXTRA, MMA, B>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  ua_blend_fast_kernel<LC, RGB, ENT, EXTRA, MMA, B><<<(unsigned)a.total_tiles, 256, sm, s>>>(a);
}

// entropy-only renders (select_nbv without RGB) stage no colours: 384-entry
// batches (fewer barriers; measured 128/192/256/384: 3347/3410/3440/3488 views/s)
template <int LC, bool RGB, bool ENT, bool EXTRA, bool MMA>
void launch_fast_kernel(const UaBlendArgs& a, cudaStream_t s) {
  launch_fast_kernel_b<LC, RGB, ENT, EXTRA, MMA, MMA ? kFastBatchMma : (RGB ? kFastBatch : 384)>(a, s);
}

// Colour path: the tensor-core GEMM by default, GAVIS_UA_COLOR=ffma selects the
// packed-FFMA dot products (A/B measurements).
inline bool colour_mma() {
  static const bool mma = [] {
    const char* e = std::getenv("GAVIS_UA_COLOR");
    return !(e && e[0] == 'f');
  }();
  return mma;
}

template <int LC, bool RGB, bool ENT, bool EXTRA>
void launch_fast_one(const UaBlendArgs& a, cudaStream_t s) {
  if (RGB && a.scene.colors_split)  // built when colour_mma() (ua_colors_split_bytes)
    launch_fast_kernel<LC, RGB, ENT, EXTRA, true>(a, s);
  else
    launch_fast_kernel<LC, RGB, ENT, EXTRA, false>(a, s);
}

template <int LC, bool EXTRA>
void launch_fast_lc(const UaBlendArgs& a, cudaStream_t s) {
  if (a.do_rgb && a.do_ent)
    launch_fast_one<LC, true, true, EXTRA>(a, s);
  else if (a.do_rgb)
    launch_fast_one<LC, true, false, EXTRA>(a, s);
  else if (a.do_ent)
    launch_fast_one<LC, false, true, EXTRA>(a, s);
}

template <int LC>
void launch_redo_lc(const UaBlendArgs& a, cudaStream_t s) {
  // one-warp blocks: they fit beside the next batch's blend CTAs (3 x 20k
  // registers per SM leave room for one redo warp), so the redo of batch k runs
  // on the side stream underneath batch k+1 instead of holding whole SMs
  const unsigned grid = 148 * 32;
  if (a.do_rgb && a.do_ent)
    ua_redo_kernel<LC, true, true><<<grid, 32, 0, s>>>(a);
  else if (a.do_rgb)
    ua_redo_kernel<LC, true, false><<<grid, 32, 0, s>>>(a);
  else if (a.do_ent)
    ua_redo_kernel<LC, false, true><<<grid, 32, 0, s>>>(a);
}

}  // namespace

bool ua_fast_supported(int tile_size, double amax) { return tile_size == 16 && amax <= 0.999; }

void launch_ua_blend_fast(const UaBlendArgs& a, cudaStream_t s) {
  if (a.total_tiles == 0) return;
  const bool extra = a.depth || a.edepth || a.rgb_contrib || a.ent_contrib || a.corr_lambda > 0.0;
  switch (a.scene.color_degree) {
#define GAVIS_FAST_LC(L)                \
  case L:                               \
    if (extra)                          \
      launch_fast_lc<L, true>(a, s);    \
    else                                \
      launch_fast_lc<L, false>(a, s);   \
    break;
    GAVIS_FAST_LC(0)
    GAVIS_FAST_LC(1)
    GAVIS_FAST_LC(2)
    GAVIS_FAST_LC(3)
#undef GAVIS_FAST_LC
    default: break;
  }
}

bool ua_exact_mma_supported(const UaBlendArgs& a) {
  return a.tile_size == 16 && a.do_rgb && a.scene.colors_split != nullptr && colour_mma();
}

void launch_ua_blend_exact_mma(const UaBlendArgs& a, cudaStream_t s) {
  if (a.total_tiles == 0) return;
  const bool extra = a.depth || a.edepth || a.rgb_contrib || a.ent_contrib || a.corr_lambda > 0.0;
  switch (a.scene.color_degree) {
#define GAVIS_EXACT_LC(L)                 \
  case L:                                 \
    if (extra)                            \
      launch_exact_mma_lc<L, true>(a, s); \
    else                                  \
      launch_exact_mma_lc<L, false>(a, s); \
    break;
    GAVIS_EXACT_LC(0)
    GAVIS_EXACT_LC(1)
    GAVIS_EXACT_LC(2)
    GAVIS_EXACT_LC(3)
#undef GAVIS_EXACT_LC
    default: break;
  }
}

void launch_ua_redo(const UaBlendArgs& a, cudaStream_t s) {
  if (a.total_tiles == 0) return;
  switch (a.scene.color_degree) {
    case 0: launch_redo_lc<0>(a, s); break;
    case 1: launch_redo_lc<1>(a, s); break;
    case 2: launch_redo_lc<2>(a, s); break;
    case 3: launch_redo_lc<3>(a, s); break;
    default: break;
  }
}

void launch_score_image(const DevCam* cams, int V, const double* entropy, const double* edepth,
                        double corr_lambda, double* partial, double* scores, cudaStream_t s) {
  if (V == 0) return;
  score_image_kernel<<<dim3(kScoreChunks, V), 256, 0, s>>>(cams, entropy, edepth, corr_lambda, partial);
  score_fold_kernel<<<V, 32, 0, s>>>(partial, scores);
}

int score_partials_per_view() { return kScoreChunks; }

size_t ua_colors_split_bytes(const SceneDev& scene) {
  if (!colour_mma() || scene.color_degree < 0 || scene.color_degree > 3) return 0;
  return sizeof(uint32_t) * kColWords * (size_t)std::max<int64_t>(scene.n, 1);
}

void launch_split_colors(const SceneDev& scene, uint4* out, cudaStream_t s) {
  if (scene.n == 0) return;
  const int64_t work = scene.n * 12;
  const unsigned grid = (unsigned)((work + 255) / 256);
  uint32_t* o = reinterpret_cast<uint32_t*>(out);
  switch (scene.color_degree) {
    case 0: split_colors_kernel<0><<<grid, 256, 0, s>>>(scene.colors, scene.n, o); break;
    case 1: split_colors_kernel<1><<<grid, 256, 0, s>>>(scene.colors, scene.n, o); break;
    case 2: split_colors_kernel<2><<<grid, 256, 0, s>>>(scene.colors, scene.n, o); break;
    case 3: split_colors_kernel<3><<<grid, 256, 0, s>>>(scene.colors, scene.n, o); break;
    default: break;
  }
}

namespace {
__global__ void add_count_kernel(unsigned long long* total, const uint32_t* count) { *total += *count; }
}  // namespace

void launch_add_count(unsigned long long* total, const uint32_t* count, cudaStream_t s) {
  add_count_kernel<<<1, 1, 0, s>>>(total, count);
}

}  // namespace gavis
