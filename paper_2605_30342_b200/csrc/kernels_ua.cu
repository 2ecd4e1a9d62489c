// kernels_ua.cu -- fused uncertainty-aware render (K7) and score reduction (K8).
//
// K7 fuses, per pixel and over the same sorted tile list:
//   * rasterize's RGB track (R/include/gavis/raster.hpp:191-229): plain alpha,
//     w = alpha*T, rgb += w*clamp(SH colour at the pixel ray), T *= 1-alpha,
//     stop once T < cutoff;
//   * render_entropy_core's entropy track (uncertainty.hpp:177-236):
//     alpha* = clamp(A*alpha + B), w = alpha*T*, s = w*v,
//     H += s(-ln s + 1/2 ln|Qc| + C_H), w0 += w(1-v), T* *= 1-alpha*, stop once
//     T* < cutoff; afterwards H += w0(-ln w0 + 1/2 ln|Q0| + C_H) (:224-225).
// The two tracks share the splat's alpha but terminate independently; a pixel
// leaves the loop when both are done.
//
// Schedules:
//   * ua_blend_ilp_kernel (16x16 tiles, default): 256 threads, one pixel each,
//     warp pre-filter of the tile list, list entries walked two at a time in
//     straight-line code (fp64 instruction-level parallelism).
//   * ua_blend_tile2_kernel (16x16 tiles): 128 threads, two pixels per thread.
//   * ua_blend_kernel (any tile size): 256 threads, one pixel each, in rounds.
// The SH colour dot products run as packed fp32x2 FMAs (FFMA2, sm_100) over
// coefficient pairs; colour rows are padded to an even length on upload.
// Per-tile entropy partials feed K8, which folds them in tile order into the
// image score (image_entropy, uncertainty.hpp:264-272).
#include "fast_math.cuh"
#include "kernels.h"

#include <cstdlib>

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

template <int LC, bool RGB, bool ENT>
__device__ __forceinline__ void pixel_init(Pixel<LC>& P, const DevCam& c, int px, int py,
                                           bool inside) {
  constexpr int NB = Col<LC>::NB;
  if (RGB) {
    // CameraView::pixel_ray (model.hpp:83-86) + eval_real_sh_block at the ray.
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
    for (int i = 0; i < Col<LC>::NP; ++i) P.bp[i] = make_float2((float)bd[2 * i], (float)bd[2 * i + 1]);
  }
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

// alpha of splat e at the pixel (splat_alpha, raster.hpp:101-108).
__device__ __forceinline__ double splat_alpha(const GeoRec& e, double cxp, double cyp, double amax) {
  const double dx = cxp - e.mx;
  const double dy = cyp - e.my;
  const double q = e.ca * dx * dx + e.cb2 * dx * dy + e.cc * dy * dy;
  double al = 0.0;  // q > kQSkip: alpha < 2^-54, T bit-identical (fast_math.cuh)
  if (q <= kQSkip) {
    al = (double)e.opacity * exp_neg(-0.5 * q);
    al = al > amax ? amax : al;
  }
  return al;
}

// RGB track update given alpha and (if w > 0) the colour (raster.hpp:209-221).
// EXTRA: depth and contributor counts (only when an output asks for them).
template <int LC, bool EXTRA>
__device__ __forceinline__ void rgb_step(Pixel<LC>& P, double al, double depth, const float2* col2,
                                         double cutoff) {
  if (EXTRA) ++P.n_rgb;
  const double w = al * P.T;
  if (w > 0.0) {
    float c0, c1, c2;
    sh_color<LC>(col2, P.bp, c0, c1, c2);
    P.rgb0 += w * (double)c0;
    P.rgb1 += w * (double)c1;
    P.rgb2 += w * (double)c2;
    if (EXTRA) P.dep += w * depth;
  }
  P.T *= 1.0 - al;
  if (P.T < cutoff) P.rgb_done = true;
}

// Entropy track update (uncertainty.hpp:198-222).
template <int LC, bool EXTRA>
__device__ __forceinline__ void ent_step(Pixel<LC>& P, double al, double depth, const UaRec& u,
                                         double amax, double cutoff, double hl_qc) {
  if (EXTRA) ++P.n_ent;
  double as = u.A * al + u.B;
  as = as < 0.0 ? 0.0 : (amax < as ? amax : as);
  const double w = as * P.Te;
  const double s = w * u.v;
  if (s > 0.0) P.H += s * (-log_pos(s) + u.hl + kGaussEntropy);
  P.w0 += w * (1.0 - u.v);
  if (EXTRA) P.edep += w * depth;
  P.Te *= 1.0 - as;
  if (P.Te < cutoff) P.ent_done = true;
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

// Per-pixel contribution to image_entropy (uncertainty.hpp:264-278): H, or with
// the correlation hook H - H exp(-d / lambda), d the entropy-track depth.
template <int LC>
__device__ __forceinline__ double score_term(const Pixel<LC>& P, const UaBlendArgs& a) {
  if (a.corr_lambda > 0.0) return P.H - P.H * exp(-P.edep / a.corr_lambda);
  return P.H;
}

template <int LC, bool RGB, bool ENT>
struct Stage {
  static constexpr size_t bytes(int batch) {
    return (size_t)batch * (sizeof(GeoRec) + sizeof(int4) + (ENT ? sizeof(UaRec) : 0) +
                            (RGB ? sizeof(float) * Col<LC>::STRIDE : 0));
  }
};

// Stage entries [base, base+n) of the tile list into shared memory.
template <int LC, bool RGB, bool ENT>
__device__ __forceinline__ void stage_batch(const UaBlendArgs& a, const GeoRec* geo, const UaRec* uar,
                                            uint32_t base, int n, GeoRec* s_geo, int4* s_rect,
                                            UaRec* s_ua, float* s_col) {
  constexpr int V4 = Col<LC>::STRIDE / 4;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const uint32_t g = a.vals[base + j];
    const GeoRec r = geo[g];
    s_geo[j] = r;
    s_rect[j] = cover_rect4(r.cov_x, r.cov_y);
    if (ENT) s_ua[j] = uar[g];
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

// ---------------------------------------------------------------------------
// 16x16 tiles, 128 threads, two pixels per thread.
template <int LC, bool RGB, bool ENT, bool EXTRA>
__global__ void __launch_bounds__(128, 5) ua_blend_tile2_kernel(UaBlendArgs a) {
  constexpr int CS = Col<LC>::STRIDE;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  GeoRec* s_geo = reinterpret_cast<GeoRec*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + kBatch * sizeof(GeoRec));
  UaRec* s_ua = reinterpret_cast<UaRec*>(s_dyn + kBatch * (sizeof(GeoRec) + sizeof(int4)));
  float* s_col = reinterpret_cast<float*>(s_dyn + kBatch * (sizeof(GeoRec) + sizeof(int4) +
                                                            (ENT ? sizeof(UaRec) : 0)));
  __shared__ double s_red[4];
  load_math_tables();

  const double amax = a.amax, cutoff = a.cutoff, hl_qc = a.hl_qc;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;

  const int px = tx * 16 + (warp & 1) * 8 + (lane & 7);
  const int py0 = ty * 16 + (warp >> 1) * 8 + (lane >> 3);
  const int py1 = py0 + 4;
  const int bx0 = tx * 16 + (warp & 1) * 8, by0 = ty * 16 + (warp >> 1) * 8;
  const bool in0 = px < c.width && py0 < c.height;
  const bool in1 = px < c.width && py1 < c.height;
  const double cxp = px + 0.5, cyp0 = py0 + 0.5, cyp1 = py1 + 0.5;
  Pixel<LC> P0, P1;
  pixel_init<LC, RGB, ENT>(P0, c, px, py0, in0);
  pixel_init<LC, RGB, ENT>(P1, c, px, py1, in1);

  for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
    const bool live = !(P0.rgb_done && P0.ent_done && P1.rgb_done && P1.ent_done);
    if (__syncthreads_count(live) == 0) break;
    const int n = min((uint32_t)kBatch, rg.y - base);
    stage_batch<LC, RGB, ENT>(a, geo, uar, base, n, s_geo, s_rect, s_ua, s_col);
    __syncthreads();
    if (__all_sync(0xffffffffu, !live)) continue;
    // warp pre-filter: one lane per entry tests the entry's coverage rectangle
    // against the warp's 8x8 pixel block; only hits are walked (in list order).
    for (int j0 = 0; j0 < n; j0 += 32) {
      bool hit = false;
      if (j0 + lane < n) {
        const int4 r = s_rect[j0 + lane];
        hit = r.x <= bx0 + 7 && r.x + r.y >= bx0 && r.z <= by0 + 7 && r.z + r.w >= by0;
      }
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      while (hits != 0u) {
      const int j = j0 + __ffs(hits) - 1;
      hits &= hits - 1u;
      const int4 rr = s_rect[j];
      const bool c0 = !(P0.rgb_done && P0.ent_done) && in_rect4(rr, px, py0);
      const bool c1 = !(P1.rgb_done && P1.ent_done) && in_rect4(rr, px, py1);
      if (!(c0 || c1)) continue;
      const GeoRec& e = s_geo[j];
      const float2* col2 = reinterpret_cast<const float2*>(s_col + j * CS);
      if (c0) {
        const double al = splat_alpha(e, cxp, cyp0, amax);
        if (RGB && !P0.rgb_done) rgb_step<LC, EXTRA>(P0, al, e.depth, col2, cutoff);
        if (ENT && !P0.ent_done) ent_step<LC, EXTRA>(P0, al, e.depth, s_ua[j], amax, cutoff, hl_qc);
      }
      if (c1) {
        const double al = splat_alpha(e, cxp, cyp1, amax);
        if (RGB && !P1.rgb_done) rgb_step<LC, EXTRA>(P1, al, e.depth, col2, cutoff);
        if (ENT && !P1.ent_done) ent_step<LC, EXTRA>(P1, al, e.depth, s_ua[j], amax, cutoff, hl_qc);
      }
      }
    }
  }
  pixel_finish<LC, RGB, ENT, EXTRA>(P0, a, c, px, py0, in0);
  pixel_finish<LC, RGB, ENT, EXTRA>(P1, a, c, px, py1, in1);
  if (ENT && a.tile_score) {
    double h = (in0 ? score_term(P0, a) : 0.0) + (in1 ? score_term(P1, a) : 0.0);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if (lane == 0) s_red[warp] = h;
    __syncthreads();
    if (tid == 0) a.tile_score[gt] = ((s_red[0] + s_red[1]) + s_red[2]) + s_red[3];
  }
}

// ---------------------------------------------------------------------------
// Any tile size: 256 threads, one pixel each, pixels in rounds of 256.
template <int LC, bool RGB, bool ENT, bool EXTRA>
__global__ void __launch_bounds__(256) ua_blend_kernel(UaBlendArgs a) {
  constexpr int CS = Col<LC>::STRIDE;
  constexpr int kThreads = 256, kWarps = 8;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  GeoRec* s_geo = reinterpret_cast<GeoRec*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + kBatch * sizeof(GeoRec));
  UaRec* s_ua = reinterpret_cast<UaRec*>(s_dyn + kBatch * (sizeof(GeoRec) + sizeof(int4)));
  float* s_col = reinterpret_cast<float*>(s_dyn + kBatch * (sizeof(GeoRec) + sizeof(int4) +
                                                            (ENT ? sizeof(UaRec) : 0)));
  __shared__ double s_red[kWarps];
  load_math_tables();

  const double amax = a.amax, cutoff = a.cutoff, hl_qc = a.hl_qc;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int ts = a.tile_size;
  const int rounds = (ts * ts + kThreads - 1) / kThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;
  double tile_h = 0.0;

  for (int round = 0; round < rounds; ++round) {
    const int li = round * kThreads + tid;
    const int lx = li % ts, ly = li / ts;
    const int px = tx * ts + lx, py = ty * ts + ly;
    const bool inside = li < ts * ts && px < c.width && py < c.height;
    const double cxp = px + 0.5, cyp = py + 0.5;
    Pixel<LC> P;
    pixel_init<LC, RGB, ENT>(P, c, px, py, inside);
    for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
      const bool live = !(P.rgb_done && P.ent_done);
      if (__syncthreads_count(live) == 0) break;
      const int n = min((uint32_t)kBatch, rg.y - base);
      stage_batch<LC, RGB, ENT>(a, geo, uar, base, n, s_geo, s_rect, s_ua, s_col);
      __syncthreads();
      if (!live) continue;
      for (int j = 0; j < n; ++j) {
        if (!in_rect4(s_rect[j], px, py)) continue;
        const GeoRec& e = s_geo[j];
        const double al = splat_alpha(e, cxp, cyp, amax);
        if (RGB && !P.rgb_done)
          rgb_step<LC, EXTRA>(P, al, e.depth, reinterpret_cast<const float2*>(s_col + j * CS), cutoff);
        if (ENT && !P.ent_done) ent_step<LC, EXTRA>(P, al, e.depth, s_ua[j], amax, cutoff, hl_qc);
        if (P.rgb_done && P.ent_done) break;
      }
    }
    pixel_finish<LC, RGB, ENT, EXTRA>(P, a, c, px, py, inside);
    if (ENT && a.tile_score) {
      double h = inside ? score_term(P, a) : 0.0;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
      if (lane == 0) s_red[warp] = h;
      __syncthreads();
      if (tid == 0) {
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) sum += s_red[w];
        tile_h += sum;
      }
    }
    __syncthreads();
  }
  if (ENT && a.tile_score && tid == 0) a.tile_score[gt] = tile_h;
}

// ---------------------------------------------------------------------------
// 16x16 tiles, 256 threads, one pixel each (warp = 8x4 patch), list entries
// walked TWO AT A TIME in straight-line code. fp64 ops have an 8-cycle
// dependent latency on B200 (tools/micro/lat.cu): the alphas (exp), colours and
// logs of the two entries are independent, so the pair doubles the fp64
// instruction-level parallelism; only T, T*, rgb, H and w0 chain. Masks replace
// branches: an entry a pixel does not cover, or one past its termination, gets
// alpha = alpha* = 0, which leaves every accumulator bit-identical.
template <int LC, bool RGB, bool ENT, bool EXTRA, int BATCH = kBatch>
__global__ void __launch_bounds__(256, 3) ua_blend_ilp_kernel(UaBlendArgs a) {
  constexpr int CS = Col<LC>::STRIDE;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  GeoRec* s_geo = reinterpret_cast<GeoRec*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + BATCH * sizeof(GeoRec));
  UaRec* s_ua = reinterpret_cast<UaRec*>(s_dyn + BATCH * (sizeof(GeoRec) + sizeof(int4)));
  float* s_col = reinterpret_cast<float*>(s_dyn + BATCH * (sizeof(GeoRec) + sizeof(int4) +
                                                           (ENT ? sizeof(UaRec) : 0)));
  __shared__ double s_red[8];
  load_math_tables();

  const double amax = a.amax, cutoff = a.cutoff;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;

  const int bx0 = tx * 16 + (warp & 1) * 8, by0 = ty * 16 + (warp >> 1) * 4;
  const int px = bx0 + (lane & 7), py = by0 + (lane >> 3);
  const bool inside = px < c.width && py < c.height;
  const double cxp = px + 0.5, cyp = py + 0.5;
  Pixel<LC> P;
  pixel_init<LC, RGB, ENT>(P, c, px, py, inside);

  for (uint32_t base = rg.x; base < rg.y; base += BATCH) {
    const bool live = !(P.rgb_done && P.ent_done);
    if (__syncthreads_count(live) == 0) break;
    const int n = min((uint32_t)BATCH, rg.y - base);
    stage_batch<LC, RGB, ENT>(a, geo, uar, base, n, s_geo, s_rect, s_ua, s_col);
    __syncthreads();
    if (__all_sync(0xffffffffu, !live)) continue;
    for (int j0 = 0; j0 < n; j0 += 32) {
      bool hit = false;
      if (j0 + lane < n) {
        const int4 r = s_rect[j0 + lane];
        hit = r.x <= bx0 + 7 && r.x + r.y >= bx0 && r.z <= by0 + 3 && r.z + r.w >= by0;
      }
      unsigned hits = __ballot_sync(0xffffffffu, hit);
      while (hits != 0u) {
        const int ja = j0 + __ffs(hits) - 1;
        hits &= hits - 1u;
        const bool has_b = hits != 0u;
        const int jb = has_b ? j0 + __ffs(hits) - 1 : ja;
        if (has_b) hits &= hits - 1u;
        const bool ca = in_rect4(s_rect[ja], px, py);
        const bool cb = has_b && in_rect4(s_rect[jb], px, py);
        const GeoRec& ea = s_geo[ja];
        const GeoRec& eb = s_geo[jb];
        // alphas of both entries (splat_alpha, raster.hpp:101-108), independent chains
        const double dxa = cxp - ea.mx, dya = cyp - ea.my;
        const double dxb = cxp - eb.mx, dyb = cyp - eb.my;
        const double qa = ea.ca * dxa * dxa + ea.cb2 * dxa * dya + ea.cc * dya * dya;
        const double qb = eb.ca * dxb * dxb + eb.cb2 * dxb * dyb + eb.cc * dyb * dyb;
        const double exa = exp_neg(fmax(-0.5 * qa, -40.0));
        const double exb = exp_neg(fmax(-0.5 * qb, -40.0));
        double ala = (double)ea.opacity * exa, alb = (double)eb.opacity * exb;
        ala = qa <= kQSkip ? (ala > amax ? amax : ala) : 0.0;
        alb = qb <= kQSkip ? (alb > amax ? amax : alb) : 0.0;
        if (RGB) {
          const bool ra = ca && !P.rgb_done;
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, b0 = 0.f, b1 = 0.f, b2 = 0.f;
          sh_color<LC>(reinterpret_cast<const float2*>(s_col + ja * CS), P.bp, a0, a1, a2);
          sh_color<LC>(reinterpret_cast<const float2*>(s_col + jb * CS), P.bp, b0, b1, b2);
          const double aa = ra ? ala : 0.0;
          const double wa = aa * P.T;
          P.rgb0 += wa * (double)a0;
          P.rgb1 += wa * (double)a1;
          P.rgb2 += wa * (double)a2;
          if (EXTRA) P.dep += wa * ea.depth;
          P.T *= 1.0 - aa;
          const bool rd = P.rgb_done || (ra && P.T < cutoff);
          const bool rb = cb && !rd;
          const double ab = rb ? alb : 0.0;
          const double wb = ab * P.T;
          P.rgb0 += wb * (double)b0;
          P.rgb1 += wb * (double)b1;
          P.rgb2 += wb * (double)b2;
          if (EXTRA) {
            P.dep += wb * eb.depth;
            P.n_rgb += (int)ra + (int)rb;
          }
          P.T *= 1.0 - ab;
          P.rgb_done = rd || (rb && P.T < cutoff);
        }
        if (ENT) {
          const bool ea_on = ca && !P.ent_done;
          const UaRec& ua = s_ua[ja];
          const UaRec& ub = s_ua[jb];
          double xa = ua.A * ala + ua.B, xb = ub.A * alb + ub.B;
          xa = xa < 0.0 ? 0.0 : (amax < xa ? amax : xa);
          xb = xb < 0.0 ? 0.0 : (amax < xb ? amax : xb);
          const double asa = ea_on ? xa : 0.0;
          const double wa = asa * P.Te;
          const double sa = wa * ua.v;
          P.w0 += wa * (1.0 - ua.v);
          if (EXTRA) P.edep += wa * ea.depth;
          P.Te *= 1.0 - asa;
          const bool ed = P.ent_done || (ea_on && P.Te < cutoff);
          const bool eb_on = cb && !ed;
          const double asb = eb_on ? xb : 0.0;
          const double wb = asb * P.Te;
          const double sb = wb * ub.v;
          const double la = log_pos(sa > 0.0 ? sa : 1.0);
          const double lb = log_pos(sb > 0.0 ? sb : 1.0);
          if (sa > 0.0) P.H += sa * (-la + ua.hl + kGaussEntropy);
          if (sb > 0.0) P.H += sb * (-lb + ub.hl + kGaussEntropy);
          P.w0 += wb * (1.0 - ub.v);
          if (EXTRA) {
            P.edep += wb * eb.depth;
            P.n_ent += (int)ea_on + (int)eb_on;
          }
          P.Te *= 1.0 - asb;
          P.ent_done = ed || (eb_on && P.Te < cutoff);
        }
      }
    }
  }
  pixel_finish<LC, RGB, ENT, EXTRA>(P, a, c, px, py, inside);
  if (ENT && a.tile_score) {
    double h = inside ? score_term(P, a) : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xffffffffu, h, off);
    if (lane == 0) s_red[warp] = h;
    __syncthreads();
    if (tid == 0) {
      double sum = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sum += s_red[w];
      a.tile_score[gt] = sum;
    }
  }
}

// K8: image score per view = fold of its per-tile partials in tile order, one warp
// per view (lane-contiguous chunks, then a fixed shuffle tree).
__global__ void score_kernel(const DevCam* cams, int V, const double* tile_score, double* scores) {
  const int v = blockIdx.x;
  const int lane = threadIdx.x;
  const DevCam& c = cams[v];
  const int64_t nt = (int64_t)c.tiles_x * c.tiles_y;
  const int64_t lo = nt * lane / 32, hi = nt * (lane + 1) / 32;
  double sum = 0.0;
  for (int64_t i = lo; i < hi; ++i) sum += tile_score[c.tile_base + i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if (lane == 0) scores[v] = sum;
}

template <class K>
void set_smem(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int LC, bool RGB, bool ENT, bool EXTRA>
void launch_one(const UaBlendArgs& a, cudaStream_t s) {
  const size_t smem = Stage<LC, RGB, ENT>::bytes(kBatch);
  static const int choice = [] {
    const char* e = getenv("GAVIS_UA_KERNEL");
    return e ? atoi(e) : 0;
  }();
  // default for 16x16 tiles: the entry-pair (ILP) kernel; GAVIS_UA_KERNEL=3 selects
  // the two-pixel kernel, =1 the generic per-pixel kernel (A/B measurements).
  // (batch 192: fewer block barriers per tile list than 128; 3 CTAs of 58 KB fit)
  if (a.tile_size == 16 && (choice == 0 || choice == 2)) {
    constexpr int kIlpBatch = 192;
    const size_t sm = Stage<LC, RGB, ENT>::bytes(kIlpBatch);
    static bool configured = false;
    if (!configured) set_smem(ua_blend_ilp_kernel<LC, RGB, ENT, EXTRA, kIlpBatch>, sm);
    configured = true;
    ua_blend_ilp_kernel<LC, RGB, ENT, EXTRA, kIlpBatch><<<(unsigned)a.total_tiles, 256, sm, s>>>(a);
    return;
  }
  if (a.tile_size == 16 && choice == 3) {
    static bool configured = false;
    if (!configured) {
      set_smem(ua_blend_tile2_kernel<LC, RGB, ENT, EXTRA>, smem);
      configured = true;
    }
    ua_blend_tile2_kernel<LC, RGB, ENT, EXTRA><<<(unsigned)a.total_tiles, 128, smem, s>>>(a);
    return;
  }
  static bool configured = false;
  if (!configured) {
    set_smem(ua_blend_kernel<LC, RGB, ENT, EXTRA>, smem);
    configured = true;
  }
  ua_blend_kernel<LC, RGB, ENT, EXTRA><<<(unsigned)a.total_tiles, 256, smem, s>>>(a);
}

template <int LC, bool EXTRA>
void launch_lc_x(const UaBlendArgs& a, cudaStream_t s) {
  if (a.do_rgb && a.do_ent)
    launch_one<LC, true, true, EXTRA>(a, s);
  else if (a.do_rgb)
    launch_one<LC, true, false, EXTRA>(a, s);
  else if (a.do_ent)
    launch_one<LC, false, true, EXTRA>(a, s);
}

template <int LC>
void launch_lc(const UaBlendArgs& a, cudaStream_t s) {
  const bool extra = a.depth || a.edepth || a.rgb_contrib || a.ent_contrib || a.corr_lambda > 0.0;
  if (extra)
    launch_lc_x<LC, true>(a, s);
  else
    launch_lc_x<LC, false>(a, s);
}

}  // namespace

int ua_score_parts(int /*tile_size*/) { return 1; }

void launch_ua_blend(const UaBlendArgs& a, cudaStream_t s) {
  if (a.total_tiles == 0) return;
  switch (a.scene.color_degree) {
    case 0: launch_lc<0>(a, s); break;
    case 1: launch_lc<1>(a, s); break;
    case 2: launch_lc<2>(a, s); break;
    case 3: launch_lc<3>(a, s); break;
    default: break;
  }
}

void launch_score(const DevCam* cams, int V, int parts, const double* tile_score, double* scores,
                  cudaStream_t s) {
  (void)parts;
  if (V == 0) return;
  score_kernel<<<V, 32, 0, s>>>(cams, V, tile_score, scores);
}

}  // namespace gavis
