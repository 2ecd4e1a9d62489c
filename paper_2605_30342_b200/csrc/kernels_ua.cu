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
// leaves the loop when both are done, a CTA when all its pixels are.
// Per-tile entropy partials feed K8, which folds them in tile order into the
// image score (image_entropy, uncertainty.hpp:264-272).
#include "fast_math.cuh"
#include "kernels.h"

namespace gavis {

namespace {

constexpr int kThreads = 256;
constexpr int kBatch = 128;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ int find_view(const DevCam* cams, int V, int64_t tile) {
  int v = 0;
  while (v + 1 < V && cams[v + 1].tile_base <= tile) ++v;
  return v;
}

__device__ __forceinline__ void tile_pixel(int ts, int tid, int round, int& lx, int& ly) {
  if (ts == 16) {
    const int w = tid >> 5, lane = tid & 31;
    lx = (w & 1) * 8 + (lane & 7);
    ly = (w >> 1) * 4 + (lane >> 3);
  } else {
    const int li = round * kThreads + tid;
    lx = li % ts;
    ly = li / ts;
  }
}

template <int LC>
struct ColorSmem {
  static constexpr int NB = (LC + 1) * (LC + 1);
  static constexpr int STRIDE = ((3 * NB + 3) / 4) * 4;
};

template <int LC, bool RGB, bool ENT>
__global__ void __launch_bounds__(kThreads) ua_blend_kernel(UaBlendArgs a) {
  constexpr int NB = ColorSmem<LC>::NB;
  constexpr int CS = ColorSmem<LC>::STRIDE;
  __shared__ GeoRec s_geo[kBatch];
  __shared__ UaRec s_ua[ENT ? kBatch : 1];
  __shared__ __align__(16) float s_col[RGB ? kBatch * CS : 4];
  __shared__ double s_red[kWarps];
  __shared__ MathSmem s_math;
  load_math_tables(&s_math);

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
  const float4* colors4 = reinterpret_cast<const float4*>(a.scene.colors);
  double tile_h = 0.0;

  for (int round = 0; round < rounds; ++round) {
    int lx, ly;
    tile_pixel(ts, tid, round, lx, ly);
    const int px = tx * ts + lx, py = ty * ts + ly;
    const bool inside = lx < ts && ly < ts && px < c.width && py < c.height &&
                        (ts == 16 || round * kThreads + tid < ts * ts);
    const double cxp = px + 0.5, cyp = py + 0.5;

    float basis[NB];
    if (RGB) {
      // CameraView::pixel_ray (model.hpp:83-86) + eval_real_sh_block at the ray.
      const double dc0 = (cxp - c.cx) / c.fx, dc1 = (cyp - c.cy) / c.fy, dc2 = 1.0;
      const double r0 = c.R[0] * dc0 + c.R[1] * dc1 + c.R[2] * dc2;
      const double r1 = c.R[3] * dc0 + c.R[4] * dc1 + c.R[5] * dc2;
      const double r2 = c.R[6] * dc0 + c.R[7] * dc1 + c.R[8] * dc2;
      const double n2 = r0 * r0 + r1 * r1 + r2 * r2;
      const double nn = n2 > 0.0 ? sqrt(n2) : 1.0;
      double bd[NB];
      eval_sh<LC>(r0 / nn, r1 / nn, r2 / nn, bd);
#pragma unroll
      for (int i = 0; i < NB; ++i) basis[i] = (float)bd[i];
    }

    double T = 1.0, rgb0 = 0.0, rgb1 = 0.0, rgb2 = 0.0, dep = 0.0;
    double Te = 1.0, H = 0.0, w0 = 0.0, edep = 0.0;
    bool rgb_done = !(RGB && inside);
    bool ent_done = !(ENT && inside);
    int32_t n_rgb = 0, n_ent = 0;

    for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
      if (__syncthreads_count(!(rgb_done && ent_done)) == 0) break;
      const int n = min((uint32_t)kBatch, rg.y - base);
      for (int j = tid; j < n; j += kThreads) {
        const uint32_t g = a.vals[base + j];
        s_geo[j] = geo[g];
        if (ENT) s_ua[j] = uar[g];
      }
      if (RGB) {
        constexpr int V4 = CS / 4;
        for (int k = tid; k < n * V4; k += kThreads) {
          const int j = k / V4, q = k - j * V4;
          const uint32_t g = a.vals[base + j];
          reinterpret_cast<float4*>(s_col)[k] = colors4[(int64_t)g * V4 + q];
        }
      }
      __syncthreads();
      if (!(rgb_done && ent_done)) {
        for (int j = 0; j < n; ++j) {
          const GeoRec& e = s_geo[j];
          if (px < cov_lo(e.cov_x) || px > cov_hi(e.cov_x) || py < cov_lo(e.cov_y) ||
              py > cov_hi(e.cov_y))
            continue;
          const double dx = cxp - e.mx;
          const double dy = cyp - e.my;
          const double q = e.ca * dx * dx + e.cb2 * dx * dy + e.cc * dy * dy;
          double al = 0.0;  // q > kQSkip: alpha < 2^-54, T bit-identical (fast_math.cuh)
          if (q <= kQSkip) {
            al = (double)e.opacity * exp_neg(-0.5 * q, &s_math);
            al = al > a.amax ? a.amax : al;
          }
          if (RGB && !rgb_done) {
            ++n_rgb;
            const double w = al * T;
            if (w > 0.0) {
              const float* col = s_col + j * CS;
              float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
              for (int i = 0; i < NB; ++i) {
                c0 = __fmaf_rn(col[i], basis[i], c0);
                c1 = __fmaf_rn(col[NB + i], basis[i], c1);
                c2 = __fmaf_rn(col[2 * NB + i], basis[i], c2);
              }
              c0 = fminf(fmaxf(c0, 0.f), 1.f);
              c1 = fminf(fmaxf(c1, 0.f), 1.f);
              c2 = fminf(fmaxf(c2, 0.f), 1.f);
              rgb0 += w * (double)c0;
              rgb1 += w * (double)c1;
              rgb2 += w * (double)c2;
              dep += w * e.depth;
            }
            T *= 1.0 - al;
            if (T < a.cutoff) rgb_done = true;
          }
          if (ENT && !ent_done) {
            ++n_ent;
            const UaRec& u = s_ua[j];
            double as = u.A * al + u.B;
            as = as < 0.0 ? 0.0 : (a.amax < as ? a.amax : as);
            const double w = as * Te;
            const double s = w * u.v;
            if (s > 0.0) H += s * (-log_pos(s, &s_math) + a.hl_qc + kGaussEntropy);
            w0 += w * u.omv;
            edep += w * e.depth;
            Te *= 1.0 - as;
            if (Te < a.cutoff) ent_done = true;
          }
          if (rgb_done && ent_done) break;
        }
      }
    }
    if (ENT && w0 > 0.0) H += w0 * (-log_pos(w0, &s_math) + a.hl_q0 + kGaussEntropy);
    if (inside) {
      const int64_t pix = c.pix_base + (int64_t)py * c.width + px;
      if (RGB) {
        if (a.rgb) {
          a.rgb[pix * 3 + 0] = rgb0;
          a.rgb[pix * 3 + 1] = rgb1;
          a.rgb[pix * 3 + 2] = rgb2;
        }
        if (a.depth) a.depth[pix] = dep;
        if (a.trans) a.trans[pix] = T;
        if (a.rgb_contrib) a.rgb_contrib[pix] = n_rgb;
      }
      if (ENT) {
        if (a.entropy) a.entropy[pix] = H;
        if (a.w0) a.w0[pix] = w0;
        if (a.edepth) a.edepth[pix] = edep;
        if (a.ent_contrib) a.ent_contrib[pix] = n_ent;
      }
    }
    if (ENT && a.tile_score) {
      double h = inside ? H : 0.0;
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

// K8: image score per view = fold of its tile partials in tile order, one warp
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

template <int LC>
void launch_lc(const UaBlendArgs& a, cudaStream_t s) {
  const unsigned grid = (unsigned)a.total_tiles;
  if (a.do_rgb && a.do_ent)
    ua_blend_kernel<LC, true, true><<<grid, kThreads, 0, s>>>(a);
  else if (a.do_rgb)
    ua_blend_kernel<LC, true, false><<<grid, kThreads, 0, s>>>(a);
  else if (a.do_ent)
    ua_blend_kernel<LC, false, true><<<grid, kThreads, 0, s>>>(a);
}

}  // namespace

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

void launch_score(const DevCam* cams, int V, const double* tile_score, double* scores,
                  cudaStream_t s) {
  if (V == 0) return;
  score_kernel<<<V, 32, 0, s>>>(cams, V, tile_score, scores);
}

}  // namespace gavis
