// ua_common.cuh -- device helpers shared by the UA blend kernels (K7): the fp64
// per-pixel state and steps of the exact path (kernels_ua.cu, also used by the
// certified path's fp64 redo in kernels_ua_fast.cu), the packed fp32 SH colour
// and the shared-memory staging of tile-list batches.
#pragma once

#include "alpha.cuh"
#include "fast_math.cuh"
#include "kernels.h"

namespace gavis {
namespace {

constexpr int kBatch = 128;

__device__ __forceinline__ int find_view(const DevCam* cams, int V, int64_t tile) {
  int v = 0;
  while (v + 1 < V && cams[v + 1].tile_base <= tile) ++v;
  return v;
}

template <int LC>
struct Col {
  static constexpr int NB = (LC + 1) * (LC + 1);
  static constexpr int NBP = NB + (NB & 1);      // even-padded channel row
  static constexpr int NP = NBP / 2;              // coefficient pairs per channel
  static constexpr int STRIDE = ((3 * NBP + 3) / 4) * 4;
};

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra, rb, rc, rd;
  ra = *reinterpret_cast<unsigned long long*>(&a);
  rb = *reinterpret_cast<unsigned long long*>(&b);
  rc = *reinterpret_cast<unsigned long long*>(&c);
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}

template <int LC>
struct Pixel {
  double T, rgb0, rgb1, rgb2, dep;
  double Te, H, w0, edep;
  bool rgb_done, ent_done;
  int32_t n_rgb, n_ent;
  float2 bp[Col<LC>::NP];  // SH basis at the pixel ray, as pairs
};

// SH basis at the pixel ray in fp64: CameraView::pixel_ray (model.hpp:83-86)
// + eval_real_sh_block at the ray (raster.hpp:200-201).
template <int LC>
__device__ __forceinline__ void pixel_basis_d(const DevCam& c, int px, int py, double* bd) {
  const double cxp = px + 0.5, cyp = py + 0.5;
  const double dc0 = (cxp - c.cx) / c.fx, dc1 = (cyp - c.cy) / c.fy, dc2 = 1.0;
  const double r0 = c.R[0] * dc0 + c.R[1] * dc1 + c.R[2] * dc2;
  const double r1 = c.R[3] * dc0 + c.R[4] * dc1 + c.R[5] * dc2;
  const double r2 = c.R[6] * dc0 + c.R[7] * dc1 + c.R[8] * dc2;
  const double n2 = r0 * r0 + r1 * r1 + r2 * r2;
  const double nn = n2 > 0.0 ? sqrt(n2) : 1.0;
  eval_sh<LC>(r0 / nn, r1 / nn, r2 / nn, bd);
}

// The same basis as fp32 pairs (the packed colour dot products).
template <int LC>
__device__ __forceinline__ void pixel_basis(const DevCam& c, int px, int py, float2* bp) {
  constexpr int NB = Col<LC>::NB;
  const double cxp = px + 0.5, cyp = py + 0.5;
  const double dc0 = (cxp - c.cx) / c.fx, dc1 = (cyp - c.cy) / c.fy, dc2 = 1.0;
  const double r0 = c.R[0] * dc0 + c.R[1] * dc1 + c.R[2] * dc2;
  const double r1 = c.R[3] * dc0 + c.R[4] * dc1 + c.R[5] * dc2;
  const double r2 = c.R[6] * dc0 + c.R[7] * dc1 + c.R[8] * dc2;
  const double n2 = r0 * r0 + r1 * r1 + r2 * r2;
  const double nn = n2 > 0.0 ? sqrt(n2) : 1.0;
  double bd[Col<LC>::NBP];
  eval_sh<LC>(r0 / nn, r1 / nn, r2 / nn, bd);
  if (Col<LC>::NBP != NB) bd[Col<LC>::NBP - 1] = 0.0;
#pragma unroll
  for (int i = 0; i < Col<LC>::NP; ++i) bp[i] = make_float2((float)bd[2 * i], (float)bd[2 * i + 1]);
}

template <int LC, bool RGB, bool ENT>
__device__ __forceinline__ void pixel_init(Pixel<LC>& P, const DevCam& c, int px, int py,
                                           bool inside) {
  if (RGB) pixel_basis<LC>(c, px, py, P.bp);
  P.T = 1.0;
  P.rgb0 = P.rgb1 = P.rgb2 = P.dep = 0.0;
  P.Te = 1.0;
  P.H = P.w0 = P.edep = 0.0;
  P.rgb_done = !(RGB && inside);
  P.ent_done = !(ENT && inside);
  P.n_rgb = P.n_ent = 0;
}

// SH colour of one splat at one pixel ray, clamped to [0,1] (model.hpp:49-62):
// packed pairs of coefficients, even/odd partial sums folded at the end.
template <int LC>
__device__ __forceinline__ void sh_color(const float2* col2, const float2* bp, float& c0, float& c1,
                                         float& c2) {
  constexpr int NP = Col<LC>::NP;
  float2 a0 = make_float2(0.f, 0.f), a1 = a0, a2 = a0;
#pragma unroll
  for (int m = 0; m < NP; ++m) {
    a0 = ffma2(col2[m], bp[m], a0);
    a1 = ffma2(col2[NP + m], bp[m], a1);
    a2 = ffma2(col2[2 * NP + m], bp[m], a2);
  }
  c0 = __saturatef(a0.x + a0.y);
  c1 = __saturatef(a1.x + a1.y);
  c2 = __saturatef(a2.x + a2.y);
}

// ---------------------------------------------------------------------------
// fp64 arithmetic of one composited entry, shared by every exact-path kernel
// (the 16x16 entry-pair kernel, the generic kernel and the certified path's
// fp64 redo, which must agree bit for bit). The reference's expressions
// (splat_alpha raster.hpp:101-108, rasterize :209-221, render_entropy_core
// uncertainty.hpp:198-222) are evaluated in fp64 with FMA contraction where it
// saves an instruction; results agree with the unfused reference to rounding.

// One list entry as the exact blend stages it: the K1 record itself (conic
// pre-scaled by -1/2, opacity in fp64: device_common.cuh).
using ExGeo = GeoRec;
// Entropy-track constants: the K1 record itself (A, B, v, 1 - v, 1/2 ln|Q_c| + C_H,
// 1/2 ln|Q_c|; 48 bytes, 16-byte aligned: staged as a pure copy and read with
// two 128-bit and one 64-bit shared load per entry).
using ExUa = UaRec;

__device__ __forceinline__ const ExGeo& ex_geo(const GeoRec& r) { return r; }

__device__ __forceinline__ const ExUa& ex_ua(const UaRec& u) { return u; }

// compensated_alpha (uncertainty.hpp:55-59): clamp(A alpha + B, 0, alpha_max).
// LO: the lower clamp, needed only for caller-given visibilities outside [0, 1]
// (field queries give v in [0, 1], and beta, o0 in [0, 1] make A, B >= 0).
template <bool LO>
__device__ __forceinline__ double ex_astar(const ExUa& u, double al, double amax) {
  double x = fma(u.A, al, u.B);
  if (LO) x = x < 0.0 ? 0.0 : x;
  return x > amax ? amax : x;
}

// RGB track (raster.hpp:209-221): w = alpha T, rgb += w c if w > 0, T <- T (1 - alpha).
// alpha = 0 (masked entry) leaves every accumulator bit-identical. LO (inputs with
// negative opacities, where alpha < 0): the reference's `if (w > 0)` guard --
// for alpha >= 0 a w of 0 adds +0, so the guard is only needed there.
template <int LC, bool EXTRA, bool LO = false>
__device__ __forceinline__ void ex_rgb(Pixel<LC>& P, double al, double depth, float c0, float c1,
                                       float c2) {
  double w = al * P.T;
  if (LO) w = w > 0.0 ? w : 0.0;
  P.rgb0 = fma(w, (double)c0, P.rgb0);
  P.rgb1 = fma(w, (double)c1, P.rgb1);
  P.rgb2 = fma(w, (double)c2, P.rgb2);
  if (EXTRA) P.dep = fma(w, depth, P.dep);
  P.T = fma(-al, P.T, P.T);
}

// Entropy track (uncertainty.hpp:198-222) without the H term: w = a* T*,
// w0 += w (1 - v), T* <- T* (1 - a*); returns s = w v. H += s (-ln s + hl + C_H)
// is added by the caller as fma(s, hlc - ln s, H) when s > 0.
template <int LC, bool EXTRA>
__device__ __forceinline__ double ex_ent(Pixel<LC>& P, double as, const ExUa& u, double depth) {
  const double w = as * P.Te;
  P.w0 = fma(w, u.omv, P.w0);
  if (EXTRA) P.edep = fma(w, depth, P.edep);
  P.Te = fma(-as, P.Te, P.Te);
  return w * u.v;
}

// alpha of splat e at the pixel from its projection record (mixture dump).
__device__ __forceinline__ double splat_alpha(const GeoRec& r, double cxp, double cyp, double amax) {
  const ExGeo e = ex_geo(r);
  return ex_alpha(e, ex_negq(e, cxp, cyp), amax);
}

template <int LC, bool RGB, bool ENT, bool EXTRA>
__device__ __forceinline__ void pixel_finish(Pixel<LC>& P, const UaBlendArgs& a, const DevCam& c,
                                             int px, int py, bool inside) {
  if (ENT && P.w0 > 0.0) P.H += P.w0 * (-log_pos(P.w0) + a.hl_q0 + kGaussEntropy);
  if (!inside) return;
  const int64_t pix = c.pix_base + (int64_t)py * c.width + px;
  if (RGB) {
    if (a.rgb) {
      a.rgb[pix * 3 + 0] = P.rgb0;
      a.rgb[pix * 3 + 1] = P.rgb1;
      a.rgb[pix * 3 + 2] = P.rgb2;
    }
    if (EXTRA && a.depth) a.depth[pix] = P.dep;
    if (a.trans) a.trans[pix] = P.T;
    if (EXTRA && a.rgb_contrib) a.rgb_contrib[pix] = P.n_rgb;
  }
  if (ENT) {
    if (a.entropy) a.entropy[pix] = P.H;
    if (a.w0) a.w0[pix] = P.w0;
    if (EXTRA && a.edepth) a.edepth[pix] = P.edep;
    if (EXTRA && a.ent_contrib) a.ent_contrib[pix] = P.n_ent;
  }
}

template <int LC, bool RGB, bool ENT>
struct Stage {
  static constexpr size_t bytes(int batch) {
    return (size_t)batch * (sizeof(ExGeo) + sizeof(int4) + (ENT ? sizeof(ExUa) : 0) +
                            (RGB ? sizeof(float) * Col<LC>::STRIDE : 0));
  }
};

// Stage entries [base, base+n) of the tile list into shared memory as exact-path
// records (ExGeo / coverage rectangle / ExUa) and fp32 colour rows.
template <int LC, bool RGB, bool ENT>
__device__ __forceinline__ void stage_batch(const UaBlendArgs& a, const GeoRec* geo, const UaRec* uar,
                                            uint32_t base, int n, ExGeo* s_geo, int4* s_rect,
                                            ExUa* s_ua, float* s_col) {
  constexpr int V4 = Col<LC>::STRIDE / 4;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const uint32_t g = a.vals[base + j];
    const GeoRec r = geo[g];
    s_geo[j] = ex_geo(r);
    s_rect[j] = cover_rect4(r.cov_x, r.cov_y);
    if (ENT) s_ua[j] = ex_ua(uar[g]);
  }
  if (RGB) {
    const float4* colors4 = reinterpret_cast<const float4*>(a.scene.colors);
    for (int k = threadIdx.x; k < n * V4; k += blockDim.x) {
      const int j = k / V4, qd = k - j * V4;
      const uint32_t g = a.vals[base + j];
      reinterpret_cast<float4*>(s_col)[k] = __ldg(colors4 + (int64_t)g * V4 + qd);
    }
  }
}

}  // namespace
}  // namespace gavis
