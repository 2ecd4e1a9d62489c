// kernels_mixture.cu -- per-pixel mixture dump of render_entropy_core
// (R/include/gavis/uncertainty.hpp:90-102 PixelMixture, :185-230 mixtures_out).
//
// A debug/oracle output, so it runs the exact fp64 entropy track (the exact
// path's operations, ua_common.cuh), one thread per pixel, in two passes: the
// first counts the components of every pixel (composited entries with w* > 0)
// and writes w0, T* and H; after a host prefix sum the second writes the
// components {w*, v, clamp(SH colour at the pixel ray) in fp64, diag Q_c}.
#include "ua_common.cuh"

namespace gavis {

namespace {

template <int LC>
__global__ void __launch_bounds__(128) mixture_kernel(MixtureArgs a) {
  load_math_tables();
  __syncthreads();
  constexpr int NB = Col<LC>::NB;
  constexpr int NBP = Col<LC>::NBP;
  constexpr int CS = Col<LC>::STRIDE;
  const DevCam& c = *a.cam;
  const int64_t P = (int64_t)c.width * c.height;
  const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= P) return;
  const int py = (int)(pix / c.width), px = (int)(pix - (int64_t)py * c.width);
  const int64_t tile = (int64_t)(py / a.tile_size) * c.tiles_x + px / a.tile_size;
  const uint2 rg = a.ranges[tile];
  const double cxp = px + 0.5, cyp = py + 0.5;
  double basis[NB];
  pixel_basis_d<LC>(c, px, py, basis);
  double T = 1.0, H = 0.0, w0 = 0.0;
  int64_t k = 0;
  double* out = a.comps ? a.comps + 8 * a.offsets[pix] : nullptr;
  for (uint32_t j = rg.x; j < rg.y; ++j) {
    const uint32_t g = a.vals[j];
    const GeoRec e = a.geo[g];
    if (!in_rect4(cover_rect4(e.cov_x, e.cov_y), px, py)) continue;
    // the exact entropy track's operations (ex_* in ua_common.cuh)
    const double al = splat_alpha(e, cxp, cyp, a.amax);
    const ExUa u = ex_ua(a.ua[g]);
    const double as = ex_astar<true>(u, al, a.amax);  // compensated_alpha (uncertainty.hpp:55-59)
    const double w = as * T;
    const double s = w * u.v;
    if (s > 0.0) H = fma(s, u.hlc - log_blend(s), H);
    w0 = fma(w, u.omv, w0);
    if (w > 0.0) {
      if (out) {
        double* m = out + 8 * k;
        m[0] = w;
        m[1] = u.v;
        const float* col = a.scene.colors + (int64_t)g * CS;
        for (int ch = 0; ch < 3; ++ch) {
          double acc = 0.0;
#pragma unroll
          for (int i = 0; i < NB; ++i) acc += (double)col[ch * NBP + i] * basis[i];
          m[2 + ch] = acc < 0.0 ? 0.0 : (1.0 < acc ? 1.0 : acc);
        }
        double q0 = a.var_const, q1 = a.var_const, q2 = a.var_const;
        if (a.var) {  // sh_variance_propagation (uncertainty.hpp:63-83), camera-to-centre
          const float4 po = a.scene.pos_op[g];
          double d0 = po.x - c.pos[0], d1 = po.y - c.pos[1], d2 = po.z - c.pos[2];
          const double n2 = d0 * d0 + d1 * d1 + d2 * d2;
          if (n2 > 0.0) {
            const double nn = sqrt(n2);
            d0 /= nn;
            d1 /= nn;
            d2 /= nn;
          }
          double bv[(kMaxFieldDegree + 1) * (kMaxFieldDegree + 1)];
          eval_sh_rt(a.var_degree, d0, d1, d2, bv);
          const int nbv = (a.var_degree + 1) * (a.var_degree + 1);
          const float* vr = a.var + (int64_t)g * 3 * nbv;
          q0 = q1 = q2 = 0.0;
          for (int i = 0; i < nbv; ++i) {
            const double y2 = bv[i] * bv[i];
            q0 += y2 * (double)vr[i];
            q1 += y2 * (double)vr[nbv + i];
            q2 += y2 * (double)vr[2 * nbv + i];
          }
        }
        m[5] = q0;
        m[6] = q1;
        m[7] = q2;
      }
      ++k;
    }
    T = fma(-as, T, T);
    if (T < a.cutoff) break;
  }
  if (w0 > 0.0) H += w0 * (-log_pos(w0) + a.hl_q0 + kGaussEntropy);
  if (!out) {
    a.counts[pix] = k;
    a.prior[pix] = w0;
    a.resid[pix] = T;
    a.entropy[pix] = H;
  }
}

}  // namespace

void launch_mixtures(const MixtureArgs& a, int64_t P, cudaStream_t s) {
  if (P == 0) return;
  const unsigned grid = (unsigned)((P + 127) / 128);
  switch (a.scene.color_degree) {
    case 0: mixture_kernel<0><<<grid, 128, 0, s>>>(a); break;
    case 1: mixture_kernel<1><<<grid, 128, 0, s>>>(a); break;
    case 2: mixture_kernel<2><<<grid, 128, 0, s>>>(a); break;
    case 3: mixture_kernel<3><<<grid, 128, 0, s>>>(a); break;
    default: break;
  }
}

}  // namespace gavis
