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
// Schedules (the default fp64 kernel for 16x16 tiles with colour degree <= 3 is
// ua_blend_exact_mma_kernel, kernels_ua_fast.cu, dispatched from launch_ua_blend):
//   * ua_blend_ilp_kernel (16x16 tiles; colour degree > 3 or GAVIS_UA_COLOR=ffma):
//     256 threads, one pixel each,
//     warp pre-filter of the tile list, list entries walked two at a time in
//     straight-line code (fp64 instruction-level parallelism).
//   * ua_blend_kernel (any tile size): 256 threads, one pixel each, in rounds.
// The SH colour dot products run as packed fp32x2 FMAs (FFMA2, sm_100) over
// coefficient pairs; colour rows are padded to an even length on upload.
// The image score (image_entropy, uncertainty.hpp:264-272) folds the entropy
// image (K8, kernels_ua_fast.cu).
#include "ua_common.cuh"

#include <cstdlib>

namespace gavis {

namespace {

// ---------------------------------------------------------------------------
// Any tile size: 256 threads, one pixel each, pixels in rounds of 256.
template <int LC, bool RGB, bool ENT, bool EXTRA, bool LO>
__global__ void __launch_bounds__(256) ua_blend_kernel(UaBlendArgs a) {
  constexpr int CS = Col<LC>::STRIDE;
  constexpr int kThreads = 256;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  ExGeo* s_geo = reinterpret_cast<ExGeo*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + kBatch * sizeof(ExGeo));
  ExUa* s_ua = reinterpret_cast<ExUa*>(s_dyn + kBatch * (sizeof(ExGeo) + sizeof(int4)));
  float* s_col = reinterpret_cast<float*>(s_dyn + kBatch * (sizeof(ExGeo) + sizeof(int4) +
                                                            (ENT ? sizeof(ExUa) : 0)));
  load_math_tables();

  const double amax = a.amax, cutoff = a.cutoff;
  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int ts = a.tile_size;
  const int rounds = (ts * ts + kThreads - 1) / kThreads;
  const int tid = threadIdx.x;
  const int64_t N = a.scene.n;
  const GeoRec* geo = a.geo + (int64_t)v * N;
  const UaRec* uar = a.ua + (int64_t)v * N;

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
        const ExGeo& e = s_geo[j];
        const double al = ex_alpha(e, ex_negq(e, cxp, cyp), amax);
        if (RGB && !P.rgb_done) {
          float c0, c1, c2;
          sh_color<LC>(reinterpret_cast<const float2*>(s_col + j * CS), P.bp, c0, c1, c2);
          if (EXTRA) ++P.n_rgb;
          ex_rgb<LC, EXTRA, LO>(P, al, e.depth, c0, c1, c2);
          if (P.T < cutoff) P.rgb_done = true;
        }
        if (ENT && !P.ent_done) {
          const ExUa& u = s_ua[j];
          if (EXTRA) ++P.n_ent;
          const double sv = ex_ent<LC, EXTRA>(P, ex_astar<LO>(u, al, amax), u, e.depth);
          if (sv > 0.0) P.H = fma(sv, u.hlc - log_blend(sv), P.H);
          if (P.Te < cutoff) P.ent_done = true;
        }
        if (P.rgb_done && P.ent_done) break;
      }
    }
    pixel_finish<LC, RGB, ENT, EXTRA>(P, a, c, px, py, inside);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// 16x16 tiles, 256 threads, one pixel each (warp = 8x4 patch), list entries
// walked TWO AT A TIME in straight-line code. fp64 ops have an 8-cycle
// dependent latency on B200 (tools/micro/lat.cu): the alphas (exp), colours and
// logs of the two entries are independent, so the pair doubles the fp64
// instruction-level parallelism; only T, T*, rgb, H and w0 chain. Masks replace
// branches: an entry a pixel does not cover, or one past its termination, gets
// alpha = alpha* = 0, which leaves every accumulator bit-identical.
template <int LC, bool RGB, bool ENT, bool EXTRA, bool LO, int BATCH = kBatch>
// (entropy-only renders -- select_nbv without RGB -- fit 4 CTAs per SM in 63
// registers without spills; the FFMA-colour RGB variants need 80, 3 CTAs)
__global__ void __launch_bounds__(256, RGB ? 3 : 4) ua_blend_ilp_kernel(UaBlendArgs a) {
  constexpr int CS = Col<LC>::STRIDE;
  extern __shared__ __align__(16) unsigned char s_dyn[];
  ExGeo* s_geo = reinterpret_cast<ExGeo*>(s_dyn);
  int4* s_rect = reinterpret_cast<int4*>(s_dyn + BATCH * sizeof(ExGeo));
  ExUa* s_ua = reinterpret_cast<ExUa*>(s_dyn + BATCH * (sizeof(ExGeo) + sizeof(int4)));
  float* s_col = reinterpret_cast<float*>(s_dyn + BATCH * (sizeof(ExGeo) + sizeof(int4) +
                                                           (ENT ? sizeof(ExUa) : 0)));
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
        const ExGeo& ea = s_geo[ja];
        const ExGeo& eb = s_geo[jb];
        // alphas of both entries (splat_alpha, raster.hpp:101-108), independent chains
        const double ala = ex_alpha(ea, ex_negq(ea, cxp, cyp), amax);
        const double alb = ex_alpha(eb, ex_negq(eb, cxp, cyp), amax);
        if (RGB) {
          float a0, a1, a2, b0, b1, b2;
          sh_color<LC>(reinterpret_cast<const float2*>(s_col + ja * CS), P.bp, a0, a1, a2);
          sh_color<LC>(reinterpret_cast<const float2*>(s_col + jb * CS), P.bp, b0, b1, b2);
          const bool ra = ca && !P.rgb_done;
          ex_rgb<LC, EXTRA, LO>(P, ra ? ala : 0.0, ea.depth, a0, a1, a2);
          const bool rd = P.rgb_done || (ra && P.T < cutoff);
          const bool rb = cb && !rd;
          ex_rgb<LC, EXTRA, LO>(P, rb ? alb : 0.0, eb.depth, b0, b1, b2);
          if (EXTRA) P.n_rgb += (int)ra + (int)rb;
          P.rgb_done = rd || (rb && P.T < cutoff);
        }
        if (ENT) {
          const ExUa& ua = s_ua[ja];
          const ExUa& ub = s_ua[jb];
          const double xa = ex_astar<LO>(ua, ala, amax), xb = ex_astar<LO>(ub, alb, amax);
          const bool ea_on = ca && !P.ent_done;
          const double sa = ex_ent<LC, EXTRA>(P, ea_on ? xa : 0.0, ua, ea.depth);
          const bool ed = P.ent_done || (ea_on && P.Te < cutoff);
          const bool eb_on = cb && !ed;
          const double sb = ex_ent<LC, EXTRA>(P, eb_on ? xb : 0.0, ub, eb.depth);
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
    }
  }
  pixel_finish<LC, RGB, ENT, EXTRA>(P, a, c, px, py, inside);
}

template <class K>
void set_smem(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int LC, bool RGB, bool ENT, bool EXTRA, bool LO>
void launch_one(const UaBlendArgs& a, cudaStream_t s) {
  const size_t smem = Stage<LC, RGB, ENT>::bytes(kBatch);
  static const int choice = [] {
    const char* e = getenv("GAVIS_UA_KERNEL");
    return e ? atoi(e) : 0;
  }();
  // 16x16 tiles without the tensor-core colour: the entry-pair (ILP) kernel; GAVIS_UA_KERNEL=1 selects
  // the generic per-pixel kernel (A/B measurements). (batch 192: fewer block
  // barriers per tile list than 128; 3 CTAs of 58 KB fit)
  if (a.tile_size == 16 && choice != 1) {
    constexpr int kIlpBatch = 192;
    const size_t sm = Stage<LC, RGB, ENT>::bytes(kIlpBatch);
    static bool configured = false;
    if (!configured) set_smem(ua_blend_ilp_kernel<LC, RGB, ENT, EXTRA, LO, kIlpBatch>, sm);
    configured = true;
    ua_blend_ilp_kernel<LC, RGB, ENT, EXTRA, LO, kIlpBatch><<<(unsigned)a.total_tiles, 256, sm, s>>>(a);
    return;
  }
  static bool configured = false;
  if (!configured) {
    set_smem(ua_blend_kernel<LC, RGB, ENT, EXTRA, LO>, smem);
    configured = true;
  }
  ua_blend_kernel<LC, RGB, ENT, EXTRA, LO><<<(unsigned)a.total_tiles, 256, smem, s>>>(a);
}

template <int LC, bool EXTRA>
void launch_lc_x(const UaBlendArgs& a, cudaStream_t s) {
  // LO (the lower alpha* clamp, the RGB w > 0 guard) only for caller-given
  // visibilities outside [0, 1] or negative opacities (vis_outside_unit)
  if (a.do_rgb && a.do_ent) {
    if (a.vis_outside_unit)
      launch_one<LC, true, true, EXTRA, true>(a, s);
    else
      launch_one<LC, true, true, EXTRA, false>(a, s);
  } else if (a.do_rgb) {
    if (a.vis_outside_unit)
      launch_one<LC, true, false, EXTRA, true>(a, s);
    else
      launch_one<LC, true, false, EXTRA, false>(a, s);
  } else if (a.do_ent) {
    if (a.vis_outside_unit)
      launch_one<LC, false, true, EXTRA, true>(a, s);
    else
      launch_one<LC, false, true, EXTRA, false>(a, s);
  }
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

void launch_ua_blend(const UaBlendArgs& a, cudaStream_t s) {
  if (a.total_tiles == 0) return;
  static const int choice = [] {
    const char* e = getenv("GAVIS_UA_KERNEL");
    return e ? atoi(e) : 0;
  }();
  // RGB renders on 16x16 tiles: the fp64 blend with the tensor-core colour
  // (kernels_ua_fast.cu); GAVIS_UA_COLOR=ffma / GAVIS_UA_KERNEL=1|2 select the
  // packed-FFMA colour kernels below (A/B)
  if (choice == 0 && ua_exact_mma_supported(a)) {
    launch_ua_blend_exact_mma(a, s);
    return;
  }
  switch (a.scene.color_degree) {
    case 0: launch_lc<0>(a, s); break;
    case 1: launch_lc<1>(a, s); break;
    case 2: launch_lc<2>(a, s); break;
    case 3: launch_lc<3>(a, s); break;
    default: break;
  }
}


}  // namespace gavis
