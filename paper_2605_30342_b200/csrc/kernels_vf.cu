// kernels_vf.cu -- VF CONST blend (K6a) and SH finalize (K6b).
//
// K6a replaces the per-tile loop of single_view_visibility
// (R/include/gavis/raster.hpp:249-274): per pixel, front to back over the
// covered entries, v_k += T, c_k += 1, T *= 1 - alpha, stop once T < cutoff.
// One CTA per 16x16 tile, one thread per pixel, warps on 8x4 pixel patches.
// Entries are staged in shared memory in batches; per entry the covered lanes
// of a warp are found with a ballot and their T values summed with a
// fixed-order shuffle tree, so the per-(tile, entry) partial is deterministic.
// Partials land in the entry's ORIGINAL pair slot: pairs of one particle are
// emitted in ascending tile order, so K6b can fold them in the reference's
// tile-merge order (raster.hpp:276-285).
//
// K6b replaces the merge/average (raster.hpp:276-289) and accumulate_view
// (vfield.hpp:38-63): one thread per particle folds its pairs, divides by the
// touch count and adds v * a_l * Y_lm(d) to its SH row, views in trajectory
// order.
#include "alpha.cuh"
#include "fast_math.cuh"
#include "kernels.h"

#include <cstdlib>

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

// Pixel of thread `tid` in round `round` of a ts x ts tile. For 16x16 tiles each
// warp owns an 8x4 patch (squarer footprint -> fewer divergent lanes per splat).
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

__global__ void __launch_bounds__(kThreads) vf_blend_kernel(VfBlendArgs a) {
  __shared__ GeoRec s_geo[kBatch];
  __shared__ int4 s_rect[kBatch];
  __shared__ uint32_t s_pair[kBatch];
  __shared__ double s_sum[kWarps][kBatch];
  __shared__ int32_t s_cnt[kWarps][kBatch];
  load_math_tables();

  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int ts = a.tile_size;
  const int rounds = (ts * ts + kThreads - 1) / kThreads;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const GeoRec* geo = a.geo + (int64_t)v * a.N;

  for (int round = 0; round < rounds; ++round) {
    int lx, ly;
    tile_pixel(ts, tid, round, lx, ly);
    const int px = tx * ts + lx, py = ty * ts + ly;
    const bool inside = lx < ts && ly < ts && px < c.width && py < c.height &&
                        (ts == 16 || round * kThreads + tid < ts * ts);
    const double cxp = px + 0.5, cyp = py + 0.5;
    double T = 1.0;
    bool done = !inside;
    int32_t ncontrib = 0;

    for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
      if (__syncthreads_count(!done) == 0) break;
      const int n = min((uint32_t)kBatch, rg.y - base);
      for (int j = tid; j < n; j += kThreads) {
        const uint32_t p = a.vals[base + j];
        s_pair[j] = p;
        const GeoRec r = geo[a.pair_gid[p]];
        s_geo[j] = r;
        s_rect[j] = cover_rect4(r.cov_x, r.cov_y);
      }
      for (int k = tid; k < kWarps * kBatch; k += kThreads) {
        (&s_sum[0][0])[k] = 0.0;
        (&s_cnt[0][0])[k] = 0;
      }
      __syncthreads();
      for (int j = 0; j < n; ++j) {
        const bool cov = !done && in_rect4(s_rect[j], px, py);
        const unsigned mask = __ballot_sync(0xffffffffu, cov);
        if (mask == 0u) continue;
        double contrib = 0.0;
        if (cov) {
          const GeoRec& e = s_geo[j];
          contrib = T;  // v_k += T before the splat (raster.hpp:266)
          ++ncontrib;
          // alpha (alpha.cuh) and T (1 - alpha) in one rounding
          const double al = ex_alpha(e, ex_negq(e, cxp, cyp), a.amax);
          T = fma(-al, T, T);
          if (T < a.cutoff) done = true;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, off);
        if (lane == 0) {
          s_sum[warp][j] = contrib;
          s_cnt[warp][j] = __popc(mask);
        }
      }
      __syncthreads();
      for (int j = tid; j < n; j += kThreads) {
        double sum = 0.0;
        int32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          sum += s_sum[w][j];
          cnt += s_cnt[w][j];
        }
        if (cnt > 0) {
          const uint32_t p = s_pair[j];
          a.pair_sum[p] += sum;
          a.pair_cnt[p] += cnt;
        }
      }
    }
    if (a.contrib && inside) a.contrib[c.pix_base + (int64_t)py * c.width + px] = ncontrib;
    __syncthreads();
  }
}

// 16x16 tiles: 128 threads, two pixels per thread (rows y and y+4 of the warp's
// 8x8 block). A warp pre-filter (one lane per entry, ballot) skips entries that
// miss the block; per hit the thread folds its two pixels' T, and the warp sums
// the 32 folds exactly in fixed point: 4 + (T0 + T1) in [4, 6] carries the fold
// in its low 51 mantissa bits at 2^-50 resolution (<= 2^-51 error per fold,
// v >= 1e-4 for every contributing pixel), two 32-bit integer warp reductions
// (REDUX) add the 26-bit halves, and the 4 warps' integer totals add exactly
// at the end of the batch -- deterministic in any order, and 6 instructions
// where the fixed-order fp64 shuffle tree took 15: K6a 9.42 -> 9.25 ms per 30
// views, VF build 56.5 -> 55.6 ms (150 views). The fixed point's absolute
// resolution is relative to T >= cutoff, so it serves cutoffs >= 1e-8 (relative
// error <= 5e-8 per fold, far inside north_star's 1e-5), and its range needs
// T <= 1 (opacities >= 0, checked at scene upload); smaller cutoffs, scenes with
// negative or NaN opacities -- and GAVIS_VF_FIXED=0 -- take the fp64 shuffle
// tree (FIXED = false).
#ifndef GAVIS_VF_FIXED
#define GAVIS_VF_FIXED 1
#endif
constexpr double kVfFixedMinCutoff = 1e-8;
// register budget: the compiler's own choice (54 with the fixed-point sums);
// capping it (48 / 40) or raising it (62 / 72) measured 2-7 % slower
#ifndef GAVIS_VF_MIN_BLOCKS
#define GAVIS_VF_MIN_BLOCKS 0
#endif
#if GAVIS_VF_MIN_BLOCKS > 0
template <bool FIXED>
__global__ void __launch_bounds__(128, GAVIS_VF_MIN_BLOCKS) vf_blend_tile2_kernel(VfBlendArgs a) {
#else
template <bool FIXED>
__global__ void __launch_bounds__(128) vf_blend_tile2_kernel(VfBlendArgs a) {
#endif
  constexpr int W = 4;
  __shared__ GeoRec s_geo[kBatch];
  __shared__ int4 s_rect[kBatch];
  __shared__ uint32_t s_pair[kBatch];
  // FIXED: fixed point at 2^-50 (bits of the partials); else fp64
  __shared__ unsigned long long s_sum[W][kBatch];
  __shared__ int32_t s_cnt[W][kBatch];
  load_math_tables();

  const int64_t gt = blockIdx.x;
  const int v = find_view(a.cams, a.V, gt);
  const DevCam& c = a.cams[v];
  const int64_t t = gt - c.tile_base;
  const int tx = (int)(t % c.tiles_x), ty = (int)(t / c.tiles_x);
  const uint2 rg = a.ranges[gt];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const GeoRec* geo = a.geo + (int64_t)v * a.N;
  const double amax = a.amax, cutoff = a.cutoff;

  const int px = tx * 16 + (warp & 1) * 8 + (lane & 7);
  const int py0 = ty * 16 + (warp >> 1) * 8 + (lane >> 3), py1 = py0 + 4;
  const int bx0 = tx * 16 + (warp & 1) * 8, by0 = ty * 16 + (warp >> 1) * 8;
  const bool in0 = px < c.width && py0 < c.height, in1 = px < c.width && py1 < c.height;
  const double cxp = px + 0.5, cy0 = py0 + 0.5, cy1 = py1 + 0.5;
  double T0 = 1.0, T1 = 1.0;
  bool d0 = !in0, d1 = !in1;
  int32_t n0 = 0, n1 = 0;

  for (uint32_t base = rg.x; base < rg.y; base += kBatch) {
    if (__syncthreads_count(!(d0 && d1)) == 0) break;
    const int n = min((uint32_t)kBatch, rg.y - base);
    for (int j = tid; j < n; j += 128) {
      const uint32_t p = a.vals[base + j];
      s_pair[j] = p;
      const GeoRec r = geo[a.pair_gid[p]];
      s_geo[j] = r;
      s_rect[j] = cover_rect4(r.cov_x, r.cov_y);
    }
    for (int k = tid; k < W * kBatch; k += 128) {
      (&s_sum[0][0])[k] = 0;
      (&s_cnt[0][0])[k] = 0;
    }
    __syncthreads();
    if (!__all_sync(0xffffffffu, d0 && d1)) {
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
          const bool c0 = !d0 && in_rect4(rr, px, py0);
          const bool c1 = !d1 && in_rect4(rr, px, py1);
          const unsigned m0 = __ballot_sync(0xffffffffu, c0), m1 = __ballot_sync(0xffffffffu, c1);
          if ((m0 | m1) == 0u) continue;
          const GeoRec& e = s_geo[j];
          double contrib = 0.0;
          if (c0) {
            contrib = T0;  // v_k += T before the splat (raster.hpp:266)
            ++n0;
            const double al = ex_alpha(e, ex_negq(e, cxp, cy0), amax);
            T0 = fma(-al, T0, T0);
            d0 = T0 < cutoff;
          }
          if (c1) {
            contrib += T1;
            ++n1;
            const double al = ex_alpha(e, ex_negq(e, cxp, cy1), amax);
            T1 = fma(-al, T1, T1);
            d1 = T1 < cutoff;
          }
          if (FIXED) {
            const double y = 4.0 + contrib;  // exponent fixed: low 51 mantissa bits = contrib * 2^50
            const uint32_t ylo = (uint32_t)__double2loint(y), yhi = (uint32_t)__double2hiint(y) & 0xFFFFFu;
            const uint32_t qlo = __reduce_add_sync(0xffffffffu, ylo & 0x3FFFFFFu);  // < 32 * 2^26
            const uint32_t qhi = __reduce_add_sync(0xffffffffu, (yhi << 6) | (ylo >> 26));  // < 32 * 2^25
            if (lane == 0) s_sum[warp][j] = ((unsigned long long)qhi << 26) + qlo;
          } else {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, off);
            if (lane == 0) s_sum[warp][j] = (unsigned long long)__double_as_longlong(contrib);
          }
          if (lane == 0) s_cnt[warp][j] = __popc(m0) + __popc(m1);
        }
      }
    }
    __syncthreads();
    for (int j = tid; j < n; j += 128) {
      const double sum =
          FIXED ? (double)(s_sum[0][j] + s_sum[1][j] + s_sum[2][j] + s_sum[3][j]) * 0x1p-50
                : ((__longlong_as_double((long long)s_sum[0][j]) + __longlong_as_double((long long)s_sum[1][j])) +
                   __longlong_as_double((long long)s_sum[2][j])) +
                      __longlong_as_double((long long)s_sum[3][j]);
      const int32_t cnt = s_cnt[0][j] + s_cnt[1][j] + s_cnt[2][j] + s_cnt[3][j];
      if (cnt > 0) {
        const uint32_t p = s_pair[j];
        a.pair_sum[p] += sum;
        a.pair_cnt[p] += cnt;
      }
    }
  }
  if (a.contrib) {
    if (in0) a.contrib[c.pix_base + (int64_t)py0 * c.width + px] = n0;
    if (in1) a.contrib[c.pix_base + (int64_t)py1 * c.width + px] = n1;
  }
}

// DEG = kDegRT: any degree up to construct_field's 20, the row updated in place
// in global memory and the basis in local memory (same per-coefficient ops).
template <int DEG>
__global__ void vf_finalize_kernel(VfFinalizeArgs a, int64_t N) {
  constexpr bool RT = DEG == kDegRT;
  constexpr int NB = RT ? 1 : (DEG + 1) * (DEG + 1);
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= N) return;
  const bool virt = a.scene.virt ? a.scene.virt[g] != 0 : false;
  const float4 po = a.scene.pos_op[g];
  double row[NB];
  const bool acc = a.gamma != nullptr && !virt;
  if (acc && !RT) {
#pragma unroll
    for (int k = 0; k < NB; ++k) row[k] = a.gamma[g * NB + k];
  }
  bool touched_row = false;
  for (int v = 0; v < a.V; ++v) {
    const int64_t slot = (int64_t)v * N + g;
    double vis;
    if (a.vis_given) {
      vis = a.vis_given[g];
    } else {
      const int32_t cnt = a.counts[slot];
      double sum = 0.0;
      int64_t touch = 0;
      if (cnt > 0) {
        const int64_t o = a.offsets[slot];
        for (int k = 0; k < cnt; ++k) {
          sum += a.pair_sum[o + k];
          touch += a.pair_cnt[o + k];
        }
      }
      vis = touch > 0 ? sum / (double)touch : 0.0;
      if (a.vis_out) a.vis_out[slot] = vis;
      if (a.touch_out) a.touch_out[slot] = touch;
    }
    if (!acc || vis <= 0.0) continue;
    const DevCam& c = a.cams[v];
    double d0 = (double)po.x - c.pos[0], d1 = (double)po.y - c.pos[1], d2 = (double)po.z - c.pos[2];
    const double norm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
    if (norm < 1e-12) continue;
    d0 /= norm;
    d1 /= norm;
    d2 /= norm;
    if (RT) {
      double basis[(kMaxFieldDegreeRT + 1) * (kMaxFieldDegreeRT + 1)];
      eval_sh_rt(a.degree, d0, d1, d2, basis);
      double* gr = a.gamma + g * (int64_t)((a.degree + 1) * (a.degree + 1));
      for (int l = 0; l <= a.degree; ++l) {
        const double scale = vis * a.scales[l];
        for (int m = -l; m <= l; ++m) {
          const int idx = l * l + l + m;
          gr[idx] += scale * basis[idx];
        }
      }
      continue;
    }
    double basis[NB];
    eval_sh<(RT ? 0 : DEG)>(d0, d1, d2, basis);
#pragma unroll
    for (int l = 0; l <= (RT ? 0 : DEG); ++l) {
      const double scale = vis * a.scales[l];
#pragma unroll
      for (int m = -l; m <= l; ++m) {
        const int idx = l * l + l + m;
        row[idx] += scale * basis[idx];
      }
    }
    touched_row = true;
  }
  if (acc && touched_row && !RT) {
#pragma unroll
    for (int k = 0; k < NB; ++k) a.gamma[g * NB + k] = row[k];
  }
}

// density_control's probe product (vfield.hpp:186-190), views in order.
__global__ void density_update_kernel(double* unseen, const double* vis, int V, int64_t N,
                                      int64_t n_real, int64_t n_virtual) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_virtual) return;
  double u = unseen[k];
  for (int v = 0; v < V; ++v) u *= 1.0 - vis[(int64_t)v * N + n_real + k];
  unseen[k] = u;
}

}  // namespace

void launch_density_update(double* unseen, const double* vis, int V, int64_t N, int64_t n_real,
                           int64_t n_virtual, cudaStream_t s) {
  if (n_virtual == 0) return;
  density_update_kernel<<<(unsigned)((n_virtual + 255) / 256), 256, 0, s>>>(unseen, vis, V, N, n_real,
                                                                            n_virtual);
}

void launch_vf_blend(const VfBlendArgs& a, cudaStream_t s) {
  if (a.total_tiles == 0) return;
  static const bool generic = getenv("GAVIS_VF_GENERIC") != nullptr;
  if (a.tile_size != 16 || generic) {
    vf_blend_kernel<<<(unsigned)a.total_tiles, kThreads, 0, s>>>(a);
  } else if (GAVIS_VF_FIXED && a.fixed_sums && a.cutoff >= kVfFixedMinCutoff) {
    vf_blend_tile2_kernel<true><<<(unsigned)a.total_tiles, 128, 0, s>>>(a);
  } else {
    vf_blend_tile2_kernel<false><<<(unsigned)a.total_tiles, 128, 0, s>>>(a);
  }
}

void launch_vf_finalize(const VfFinalizeArgs& a, int64_t N, cudaStream_t s) {
  if (N == 0) return;
  const unsigned grid = (unsigned)((N + 127) / 128);
  switch (a.degree) {
    case 0: vf_finalize_kernel<0><<<grid, 128, 0, s>>>(a, N); break;
    case 1: vf_finalize_kernel<1><<<grid, 128, 0, s>>>(a, N); break;
    case 2: vf_finalize_kernel<2><<<grid, 128, 0, s>>>(a, N); break;
    case 3: vf_finalize_kernel<3><<<grid, 128, 0, s>>>(a, N); break;
    case 4: vf_finalize_kernel<4><<<grid, 128, 0, s>>>(a, N); break;
    default: vf_finalize_kernel<kDegRT><<<grid, 128, 0, s>>>(a, N); break;
  }
}

}  // namespace gavis
