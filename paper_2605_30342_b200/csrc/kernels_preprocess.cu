// kernels_preprocess.cu -- projection (K1), key emission (K3), tile ranges with
// depth-tie fix-up (K5) and the batch field query.
//
// K1 replaces project_particle / project_scene (R/include/gavis/raster.hpp:51-130)
// and, for the uncertainty render, query_visibility at the camera-to-centre
// direction (vfield.hpp:96-112 via uncertainty.hpp:251-257). One thread per
// Gaussian projects it into all V views of the batch, so the particle record
// and its SH field row are read from HBM once per batch, not once per view.
#include <math_constants.h>

#include "kernels.h"

#include <cstdio>

namespace gavis {

namespace {

constexpr int kMaxBatchViews = 64;

struct Sigma {
  double s00, s01, s02, s11, s12, s22;
  double lam;  // >= lambda_max(Sigma) (Gershgorin): bounds the screen radius before projecting
};

// GaussianParticle::covariance (model.hpp:42-45), Eigen toRotationMatrix order.
__device__ __forceinline__ Sigma covariance(float4 q, float4 sc) {
  const double w = q.x, x = q.y, y = q.z, z = q.w;
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  const double R00 = 1.0 - (tyy + tzz), R01 = txy - twz, R02 = txz + twy;
  const double R10 = txy + twz, R11 = 1.0 - (txx + tzz), R12 = tyz - twx;
  const double R20 = txz - twy, R21 = tyz + twx, R22 = 1.0 - (txx + tyy);
  const double sx = sc.x, sy = sc.y, sz = sc.z;
  const double m00 = R00 * sx, m01 = R01 * sy, m02 = R02 * sz;
  const double m10 = R10 * sx, m11 = R11 * sy, m12 = R12 * sz;
  const double m20 = R20 * sx, m21 = R21 * sy, m22 = R22 * sz;
  Sigma s;
  s.s00 = m00 * m00 + m01 * m01 + m02 * m02;
  s.s01 = m00 * m10 + m01 * m11 + m02 * m12;
  s.s02 = m00 * m20 + m01 * m21 + m02 * m22;
  s.s11 = m10 * m10 + m11 * m11 + m12 * m12;
  s.s12 = m10 * m20 + m11 * m21 + m12 * m22;
  s.s22 = m20 * m20 + m21 * m21 + m22 * m22;
  const double r0 = s.s00 + fabs(s.s01) + fabs(s.s02);
  const double r1 = fabs(s.s01) + s.s11 + fabs(s.s12);
  const double r2 = fabs(s.s02) + fabs(s.s12) + s.s22;
  s.lam = fmax(r0, fmax(r1, r2));
  return s;
}

struct Projected {
  double mx, my, c00, c01, c10, c11, depth, radius, det;
};

// project_particle (raster.hpp:51-93): returns false when culled.
__device__ __forceinline__ bool project(const DevCam& c, double px, double py, double pz,
                                        const Sigma& S, double dilation, Projected& o) {
  const double d0 = px - c.pos[0], d1 = py - c.pos[1], d2 = pz - c.pos[2];
  const double t0 = c.R[0] * d0 + c.R[3] * d1 + c.R[6] * d2;
  const double t1 = c.R[1] * d0 + c.R[4] * d1 + c.R[7] * d2;
  const double t2 = c.R[2] * d0 + c.R[5] * d1 + c.R[8] * d2;
  if (t2 < c.near_plane) return false;
  const double fx = c.fx, fy = c.fy;
  const double inv_z = 1.0 / t2;
  const double mx = c.cx + fx * t0 * inv_z;
  const double my = c.cy + fy * t1 * inv_z;
  double ux = t0 * inv_z, uy = t1 * inv_z;
  ux = ux < -c.limx ? -c.limx : (c.limx < ux ? c.limx : ux);
  uy = uy < -c.limy ? -c.limy : (c.limy < uy ? c.limy : uy);
  {
    // Frustum pre-test: lambda_max(cov2) <= lambda_max(Sigma) |J|_F^2 + dil^2, so
    // r <= rub; a particle outside the frustum by more than rub is culled below
    // anyway -- skip projecting Sigma.
    const double gx = fx * inv_z, gy = fy * inv_z;
    const double jf = gx * gx * (1.0 + ux * ux) + gy * gy * (1.0 + uy * uy);
    const double rub = 3.0 * sqrt((S.lam * jf + 2.0 * dilation * dilation) * 1.000001) + 1e-9;
    if (mx < -rub || mx > c.width + rub || my < -rub || my > c.height + rub) return false;
  }
  const double jx = ux * t2;
  const double jy = uy * t2;
  // W = R^T, cov_cam = (W Sigma) W^T ; W(r,k) = R(k,r) = c.R[k*3+r]
  const double Sg[9] = {S.s00, S.s01, S.s02, S.s01, S.s11, S.s12, S.s02, S.s12, S.s22};
  double A[9], C[9];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      A[r * 3 + k] = c.R[0 * 3 + r] * Sg[0 * 3 + k] + c.R[1 * 3 + r] * Sg[1 * 3 + k] +
                     c.R[2 * 3 + r] * Sg[2 * 3 + k];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      C[r * 3 + k] = A[r * 3 + 0] * c.R[0 * 3 + k] + A[r * 3 + 1] * c.R[1 * 3 + k] +
                     A[r * 3 + 2] * c.R[2 * 3 + k];
  const double J[6] = {fx * inv_z, 0.0, -fx * jx * inv_z * inv_z,
                       0.0, fy * inv_z, -fy * jy * inv_z * inv_z};
  double B[6];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      B[r * 3 + k] = J[r * 3 + 0] * C[0 * 3 + k] + J[r * 3 + 1] * C[1 * 3 + k] +
                     J[r * 3 + 2] * C[2 * 3 + k];
  double c00 = B[0] * J[0] + B[1] * J[1] + B[2] * J[2];
  const double c01 = B[0] * J[3] + B[1] * J[4] + B[2] * J[5];
  const double c10 = B[3] * J[0] + B[4] * J[1] + B[5] * J[2];
  double c11 = B[3] * J[3] + B[4] * J[4] + B[5] * J[5];
  c00 += dilation * dilation;
  c11 += dilation * dilation;
  const double det = c00 * c11 - c01 * c10;
  if (det <= 0.0) return false;
  const double mid = 0.5 * (c00 + c11);
  const double disc = mid * mid - det;
  const double lam_max = mid + sqrt(disc > 0.0 ? disc : 0.0);
  const double radius = 3.0 * sqrt(lam_max);
  if (mx < -radius || mx > c.width + radius || my < -radius || my > c.height + radius)
    return false;
  o.mx = mx;
  o.my = my;
  o.c00 = c00;
  o.c01 = c01;
  o.c10 = c10;
  o.c11 = c11;
  o.depth = t2;
  o.radius = radius;
  o.det = det;
  return true;
}

// query_visibility (vfield.hpp:96-112) on a register-resident row.
template <int DEG>
__device__ __forceinline__ double query_row(const double* row, int num_views, double x, double y,
                                            double z) {
  constexpr int NB = (DEG + 1) * (DEG + 1);
  double basis[NB];
  eval_sh<DEG>(x, y, z, basis);
  double vt = 0.0;
#pragma unroll
  for (int i = 0; i < NB; ++i) vt += row[i] * basis[i];
  const double p = (double)num_views;
  if (vt < 0.0) vt = 0.0;
  if (vt > p) vt = p;
  double v = 1.0 - pow(1.0 - vt / p, p);
  return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

// The same for any degree (fields above degree 4): the basis in local memory,
// the dot product in the same index order straight from the field row.
__device__ __noinline__ double query_row_rt(const double* gr, int degree, int num_views, double x,
                                            double y, double z) {
  double basis[(kMaxFieldDegreeRT + 1) * (kMaxFieldDegreeRT + 1)];
  eval_sh_rt(degree, x, y, z, basis);
  const int nb = (degree + 1) * (degree + 1);
  double vt = 0.0;
  for (int i = 0; i < nb; ++i) vt += gr[i] * basis[i];
  const double p = (double)num_views;
  if (vt < 0.0) vt = 0.0;
  if (vt > p) vt = p;
  double v = 1.0 - pow(1.0 - vt / p, p);
  return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v);
}

// Cheap visibility screen of one (view, particle): the near-plane test exactly as
// project_particle makes it (fp64, same operations), then a conservative fp32
// frustum test with the radius bound r <= 3 sqrt(lambda_max(Sigma) lambda_max(J J^T)
// + dil^2) (J C J^T <= lambda_max(C) J J^T in the Loewner order, C = W Sigma W^T
// has Sigma's spectrum; lam >= lambda_max(Sigma) by Gershgorin), inflated by 0.1 %,
// and a position margin 100x above the fp32 error: a particle it rejects is
// culled by project() as well.
__device__ __forceinline__ bool screen(const DevCam& c, double px, double py, double pz,
                                       float lam, float dil2) {
  const double d0 = px - c.pos[0], d1 = py - c.pos[1], d2 = pz - c.pos[2];
  const double t2 = c.R[2] * d0 + c.R[5] * d1 + c.R[8] * d2;
  if (t2 < c.near_plane) return false;
  const float f0 = (float)d0, f1 = (float)d1, f2 = (float)d2;
  const float t0 = __fmaf_rn((float)c.R[0], f0, __fmaf_rn((float)c.R[3], f1, (float)c.R[6] * f2));
  const float t1 = __fmaf_rn((float)c.R[1], f0, __fmaf_rn((float)c.R[4], f1, (float)c.R[7] * f2));
  const float iz = 1.f / (float)t2;
  const float ux = t0 * iz, uy = t1 * iz;
  const float fx = (float)c.fx, fy = (float)c.fy;
  const float mx = __fmaf_rn(fx, ux, (float)c.cx), my = __fmaf_rn(fy, uy, (float)c.cy);
  const float lx = (float)c.limx, ly = (float)c.limy;
  const float uxc = fminf(fmaxf(ux, -lx), lx), uyc = fminf(fmaxf(uy, -ly), ly);
  const float gx = fx * iz, gy = fy * iz;
  const float j00 = gx * gx * (1.f + uxc * uxc), j11 = gy * gy * (1.f + uyc * uyc);
  const float j01 = gx * gy * uxc * uyc;
  const float hd = 0.5f * (j00 - j11);
  const float lj = 0.5f * (j00 + j11) + sqrtf(hd * hd + j01 * j01);  // lambda_max(J J^T), no cancellation
  const float rub = 3.f * sqrtf(__fmaf_rn(lam, lj, dil2) * 1.002f);
  const float W = (float)c.width, H = (float)c.height;
  const float M = 1e-3f * (fabsf(mx) + fabsf(my) + rub + W + H) + 1e-2f;
  return !(mx + rub < -M || mx - rub > W + M || my + rub < -M || my - rub > H + M);
}

// K1. One thread per particle screens it against every view of the batch; the
// surviving (view, particle) items of a warp are compacted in shared memory and
// projected 32 at a time, so the fp64 projection runs on full warps (~10% of the
// items survive in an indoor scene; without compaction almost every warp holds
// a survivor for every view and runs the projection for all its lanes).
constexpr int kPreThreads = 128;

template <int QDEG>
__global__ void __launch_bounds__(kPreThreads) preprocess_kernel(PreprocessArgs a) {
  constexpr int kWarps = kPreThreads / 32;
  __shared__ DevCam s_cam[kMaxBatchViews];
  __shared__ uint16_t s_q[kWarps][32 * kMaxBatchViews];
  __shared__ Sigma s_sig[kPreThreads];
  for (int i = threadIdx.x; i < a.V * (int)(sizeof(DevCam) / 8); i += blockDim.x)
    reinterpret_cast<double*>(s_cam)[i] = reinterpret_cast<const double*>(a.cams)[i];
  const int64_t N = a.scene.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t wbase = (int64_t)blockIdx.x * kPreThreads + warp * 32;
  const int64_t g = wbase + lane;
  const bool valid = g < N;
  double px = 0.0, py = 0.0, pz = 0.0;
  float lam = 0.f;
  if (valid) {
    const float4 po = a.scene.pos_op[g];
    const Sigma S = covariance(a.scene.rot[g], a.scene.scale[g]);
    s_sig[threadIdx.x] = S;
    px = po.x;
    py = po.y;
    pz = po.z;
    lam = (float)S.lam;
  }
  __syncthreads();
  const float dil2 = (float)(a.dilation * a.dilation);
  const uint2 empty_rect = make_uint2(1u, 1u);  // tx0 = 1 > tx1 = 0
  int qn = 0;
  for (int v = 0; v < a.V; ++v) {
    bool surv = false;
    if (valid) {
      surv = screen(s_cam[v], px, py, pz, lam, dil2);
      if (!surv && a.cull_counts) {
        const int64_t slot = (int64_t)v * N + g;
        a.counts[slot] = 0;
        a.trect[slot] = empty_rect;
        if (a.write_culled) {
          GeoRec r = {};
          r.depth = __longlong_as_double(0x7ff8000000000000LL);  // culled
          r.cov_x = r.cov_y = kCovEmpty;
          a.geo[slot] = r;
        }
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, surv);
    if (surv) s_q[warp][qn + __popc(m & ((1u << lane) - 1u))] = (uint16_t)(lane | (v << 5));
    qn += __popc(m);
  }
  __syncwarp();
  constexpr int NBQ = (QDEG >= 0 && QDEG != kDegRT) ? (QDEG + 1) * (QDEG + 1) : 1;
  unsigned long long pairs = 0;  // this lane's tile pairs (pair_total)
  for (int k = lane; k < qn + ((32 - qn % 32) % 32); k += 32) {
    bool emit = false;
    uint32_t eslot = 0, ekey = 0;
    if (k < qn) {
    const int item = s_q[warp][k];
    const int src = item & 31, v = item >> 5;
    const int64_t gi = wbase + src;
    const float4 po = a.scene.pos_op[gi];
    const uint8_t virt = a.scene.virt ? a.scene.virt[gi] : 0;
    const Sigma S = s_sig[warp * 32 + src];
    const double qx = po.x, qy = po.y, qz = po.z;
    const DevCam& c = s_cam[v];
    const int64_t slot = (int64_t)v * N + gi;
    Projected p;
    int tx0 = 1, tx1 = 0, ty0 = 1, ty1 = 0;
    const bool ok = project(c, qx, qy, qz, S, a.dilation, p);
    int32_t count = 0;
    if (ok) {
      int x0, x1, y0, y1;
      covered_pixel_range(p.mx, p.radius, c.width, x0, x1);
      covered_pixel_range(p.my, p.radius, c.height, y0, y1);
      if (!(x0 > x1 || y0 > y1)) {
        tx0 = x0 / a.tile_size;
        tx1 = x1 / a.tile_size;
        ty0 = y0 / a.tile_size;
        ty1 = y1 / a.tile_size;
        count = (tx1 - tx0 + 1) * (ty1 - ty0 + 1);
      }
      GeoRec r;
      const double inv_det = 1.0 / p.det;
      r.mx = p.mx;
      r.my = p.my;
      // conic (a, b, c) = (c11, -c01, c00) / det, scaled by -1/2 (exact)
      r.na = -0.5 * (p.c11 * inv_det);
      r.nb = p.c01 * inv_det;
      r.nc = -0.5 * (p.c00 * inv_det);
      r.o = (double)po.w;
      r.depth = p.depth;
      r.cov_x = exact_cover(x0, x1, c.width, p.mx, p.radius);
      r.cov_y = exact_cover(y0, y1, c.height, p.my, p.radius);
      a.geo[slot] = r;
      if (a.ua) {
        double vis = 0.0;
        if (a.query_mode == kQueryGiven) {
          vis = a.vis_in[gi];
        } else if (QDEG == kDegRT && a.query_mode == kQueryField && !virt && a.num_views > 0) {
          const int nb = (a.degree + 1) * (a.degree + 1);
          const double d0 = qx - c.pos[0], d1 = qy - c.pos[1], d2 = qz - c.pos[2];
          const double norm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
          if (!(norm < 1e-12))
            vis = query_row_rt(a.gamma + gi * nb, a.degree, a.num_views, d0 / norm, d1 / norm, d2 / norm);
        } else if (QDEG >= 0 && a.query_mode == kQueryField && !virt && a.num_views > 0) {
          double row[NBQ];
          const double* gr = a.gamma + gi * NBQ;
#pragma unroll
          for (int i = 0; i < NBQ; ++i) row[i] = gr[i];
          const double d0 = qx - c.pos[0], d1 = qy - c.pos[1], d2 = qz - c.pos[2];
          const double norm = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
          if (!(norm < 1e-12))
            vis = query_row<((QDEG >= 0 && QDEG != kDegRT) ? QDEG : 0)>(row, a.num_views, d0 / norm, d1 / norm,
                                                     d2 / norm);
        }
        UaRec u;
        u.v = vis;
        u.A = vis + a.beta * (1.0 - vis);
        u.B = a.o0b * (1.0 - vis);
        u.hl = a.hl_const;
        if (a.var) {
          // sh_variance_propagation (uncertainty.hpp:63-83) at the camera-to-centre
          // direction, half log-determinant of the diagonal Q_c (:149-163).
          double d0 = qx - c.pos[0], d1 = qy - c.pos[1], d2 = qz - c.pos[2];
          const double n2 = d0 * d0 + d1 * d1 + d2 * d2;
          if (n2 > 0.0) {
            const double nn = sqrt(n2);
            d0 /= nn;
            d1 /= nn;
            d2 /= nn;
          }
          double basis[(kMaxFieldDegree + 1) * (kMaxFieldDegree + 1)];
          eval_sh_rt(a.var_degree, d0, d1, d2, basis);
          const int nbv = (a.var_degree + 1) * (a.var_degree + 1);
          const float* vr = a.var + gi * 3 * nbv;
          double q0 = 0.0, q1 = 0.0, q2 = 0.0;
          for (int i = 0; i < nbv; ++i) {
            const double y2 = basis[i] * basis[i];
            q0 += y2 * (double)vr[i];
            q1 += y2 * (double)vr[nbv + i];
            q2 += y2 * (double)vr[2 * nbv + i];
          }
          if (!(q0 > 0.0 && q1 > 0.0 && q2 > 0.0)) atomicOr(a.err_flag, 1);
          u.hl = 0.5 * (log(q0) + log(q1) + log(q2));
        }
        u.omv = 1.0 - u.v;
        u.hlc = u.hl + kGaussEntropy;
        a.ua[slot] = u;
      }
    } else if (a.write_culled) {
      GeoRec r = {};
      r.depth = __longlong_as_double(0x7ff8000000000000LL);  // culled
      r.cov_x = r.cov_y = kCovEmpty;
      a.geo[slot] = r;
    }
    a.counts[slot] = count;
    a.trect[slot] = make_uint2((uint32_t)(tx0 & 0xFFFF) | ((uint32_t)(tx1 & 0xFFFF) << 16),
                               (uint32_t)(ty0 & 0xFFFF) | ((uint32_t)(ty1 & 0xFFFF) << 16));
    pairs += (unsigned long long)count;
    if (count > 0) {
      // K2b, the item's 32-bit key: the view in the top view_bits, then the
      // leading bits of the fp32 depth rounded toward zero, sign bit dropped
      // (depth > near > 0): monotone in the fp64 depth; runs of equal keys are
      // ordered exactly by depth_order_kernel
      emit = true;
      eslot = (uint32_t)slot;
      const uint32_t db = __float_as_uint(__double2float_rz(p.depth));  // < 2^31
      ekey = ((uint32_t)v << (32 - a.view_bits)) | (db >> (a.view_bits - 1));
    }
    }
    if (a.item_slot_out) {
      const unsigned em = __ballot_sync(0xffffffffu, emit);
      if (em != 0u) {
        const int leader = __ffs(em) - 1;
        uint32_t at = 0;
        if (lane == leader) at = atomicAdd(a.n_items_out, (uint32_t)__popc(em));
        at = __shfl_sync(0xffffffffu, at, leader) + __popc(em & ((1u << lane) - 1u));
        if (emit) {
          a.item_slot_out[at] = eslot;
          a.item_key_out[at] = ekey;
        }
      }
    }
  }
  if (a.pair_total) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) pairs += __shfl_xor_sync(0xffffffffu, pairs, off);
    if (lane == 0 && pairs != 0) atomicAdd(a.pair_total, pairs);
  }
}

__global__ void emit_keys_kernel(EmitArgs a) {
  const int64_t slot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= (int64_t)a.V * a.N) return;
  const int32_t cnt = a.counts[slot];
  if (cnt == 0) return;
  const int v = (int)(slot / a.N);
  const uint32_t g = (uint32_t)(slot - (int64_t)v * a.N);
  const DevCam& c = a.cams[v];
  const uint2 tr = a.trect[slot];
  const int tx0 = tr.x & 0xFFFF, tx1 = tr.x >> 16, ty0 = tr.y & 0xFFFF, ty1 = tr.y >> 16;
  // fp32 depth rounded toward zero is monotone in the fp64 depth; runs of equal
  // fp32 keys are re-ordered by (fp64 depth, index) in ranges_kernel.
  const float df = __double2float_rz(a.geo[slot].depth);
  const uint64_t dk = (uint64_t)__float_as_uint(df);
  int64_t o = a.offsets[slot];
  for (int ty = ty0; ty <= ty1; ++ty) {
    for (int tx = tx0; tx <= tx1; ++tx) {
      const uint64_t tile = (uint64_t)(c.tile_base + (int64_t)ty * c.tiles_x + tx);
      a.keys[o] = (tile << 32) | dk;
      if (a.pair_gid) {
        a.vals[o] = (uint32_t)o;
        a.pair_gid[o] = g;
      } else {
        a.vals[o] = g;
      }
      ++o;
    }
  }
}

__device__ __forceinline__ int view_of_tile(const DevCam* cams, int V, int64_t tile) {
  int v = 0;
  while (v + 1 < V && cams[v + 1].tile_base <= tile) ++v;
  return v;
}

__global__ void ranges_kernel(RangesArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.K) return;
  const uint64_t key = a.keys[i];
  const uint64_t tile = key >> 32;
  if (i == 0 || (a.keys[i - 1] >> 32) != tile) a.ranges[tile].x = (uint32_t)i;
  if (i == a.K - 1 || (a.keys[i + 1] >> 32) != tile) a.ranges[tile].y = (uint32_t)(i + 1);
  // Depth-tie fix-up: the stable radix sort orders equal fp32 keys by particle
  // index; the reference orders by (fp64 depth, index) (raster.hpp:124-128).
  if (i + 1 < a.K && a.keys[i + 1] == key && (i == 0 || a.keys[i - 1] != key)) {
    int64_t j = i;
    while (j + 1 < a.K && a.keys[j + 1] == key) ++j;
    const int v = view_of_tile(a.cams, a.V, (int64_t)tile);
    const GeoRec* geo = a.geo + (int64_t)v * a.N;
    for (int64_t x = i + 1; x <= j; ++x) {
      const uint32_t val = a.vals[x];
      const uint32_t gx = a.pair_gid ? a.pair_gid[val] : val;
      const double dx = geo[gx].depth;
      int64_t y = x - 1;
      while (y >= i) {
        const uint32_t vy = a.vals[y];
        const uint32_t gy = a.pair_gid ? a.pair_gid[vy] : vy;
        const double dy = geo[gy].depth;
        if (dy < dx || (dy == dx && gy < gx)) break;
        a.vals[y + 1] = vy;
        --y;
      }
      a.vals[y + 1] = val;
    }
  }
}

// ---------------------------------------------------------------------------
// Depth-ordered binning (NarrowArgs): instead of sorting 64-bit (tile << 32 |
// fp32 depth) pair keys, the visible particles of each view are sorted once by
// (fp64 depth, index) -- the order of project_scene (raster.hpp:124-128) --, the
// pairs are emitted in that order and then stably radix-sorted by tile id alone
// (2-3 digit passes over 8-byte pairs instead of 6 over 12-byte pairs). Stability
// keeps the depth order inside every tile, which is exactly the reference's
// per-tile list order (splat_binning, raster.hpp:145-164).



// K2c: runs of equal 32-bit item keys ordered by (fp64 depth, index). K1 appends
// the visible items with warp-aggregated atomics, so a run arrives in scheduling
// order, not index order: a run of L items can hold O(L^2) inversions (exact
// depth ties, e.g. an axis-aligned camera facing an axis-aligned wall). Runs of
// at most kShortRun items are insertion-sorted by the thread at the run's start;
// longer runs are queued and sorted by depth_order_long_kernel, one CTA per run.
__global__ void depth_order_kernel(NarrowArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_items) return;
  const uint32_t key = a.item_key[i];
  const bool run_start = i + 1 < a.n_items && a.item_key[i + 1] == key &&
                         (i == 0 || a.item_key[i - 1] != key);
  if (!run_start) return;
  int64_t j = i;
  while (j + 1 < a.n_items && a.item_key[j + 1] == key) ++j;
  if (j - i + 1 > kShortRun) {
    const uint32_t r = atomicAdd(a.n_long, 1u);
    a.long_runs[r] = make_uint2((uint32_t)i, (uint32_t)(j - i + 1));
    return;
  }
  uint32_t* sl = a.item_slot_sorted;
  for (int64_t x = i + 1; x <= j; ++x) {
    const uint32_t sx = sl[x];
    const double dx = a.geo[sx].depth;
    int64_t y = x - 1;
    while (y >= i) {
      const uint32_t sy = sl[y];
      const double dy = a.geo[sy].depth;
      if (dy < dx || (dy == dx && sy < sx)) break;  // same view: slot order = index order
      sl[y + 1] = sy;
      --y;
    }
    sl[y + 1] = sx;
  }
}

namespace {
constexpr int kLongChunk = 2048;  // elements bitonic-sorted in shared memory per step

// (depth, slot) strict order; slots are distinct inside a run (one view).
__device__ __forceinline__ bool item_before(double da, uint32_t sa, double db, uint32_t sb) {
  return da < db || (da == db && sa < sb);
}
}  // namespace

// K2c': one CTA per long tied run (grid-stride over the queue, no host read of
// its length). Chunks of 2048 items are bitonic-sorted in shared memory, then
// merged pairwise through the scratch buffer: every item's output position is
// its index in its own half plus the number of items of the other half that
// precede it (a binary search; the keys are distinct, so no tie rule is needed).
__global__ void __launch_bounds__(256) depth_order_long_kernel(NarrowArgs a) {
  __shared__ double s_d[kLongChunk];
  __shared__ uint32_t s_s[kLongChunk];
  const int nruns = (int)*a.n_long;
  for (int r = blockIdx.x; r < nruns; r += gridDim.x) {
    const uint2 run = a.long_runs[r];
    uint32_t* const base = a.item_slot_sorted + run.x;
    uint32_t* const alt = a.scratch + run.x;
    const int L = (int)run.y;
    for (int c0 = 0; c0 < L; c0 += kLongChunk) {
      const int n = min(kLongChunk, L - c0);
      int pw = 1;
      while (pw < n) pw <<= 1;
      for (int k = threadIdx.x; k < pw; k += blockDim.x) {
        const uint32_t sl = k < n ? base[c0 + k] : 0xFFFFFFFFu;
        s_s[k] = sl;
        s_d[k] = k < n ? a.geo[sl].depth : CUDART_INF;
      }
      __syncthreads();
      for (int size = 2; size <= pw; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int k = threadIdx.x; k < pw; k += blockDim.x) {
            const int m = k ^ stride;
            if (m > k) {
              const bool up = (k & size) == 0;
              const bool swap = up ? item_before(s_d[m], s_s[m], s_d[k], s_s[k])
                                   : item_before(s_d[k], s_s[k], s_d[m], s_s[m]);
              if (swap) {
                const double td = s_d[k];
                s_d[k] = s_d[m];
                s_d[m] = td;
                const uint32_t ts = s_s[k];
                s_s[k] = s_s[m];
                s_s[m] = ts;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int k = threadIdx.x; k < n; k += blockDim.x) base[c0 + k] = s_s[k];
      __syncthreads();
    }
    uint32_t* src = base;
    uint32_t* dst = alt;
    for (int w = kLongChunk; w < L; w <<= 1) {
      for (int k = threadIdx.x; k < L; k += blockDim.x) {
        const int b0 = (k / (2 * w)) * (2 * w);
        const int mid = min(b0 + w, L), end = min(b0 + 2 * w, L);
        const uint32_t sk = src[k];
        const double dk = a.geo[sk].depth;
        const bool left = k < mid;
        int lo = left ? mid : b0, hi = left ? end : mid;  // search the other half
        const int own = left ? k - b0 : k - mid;
        while (lo < hi) {  // first element of the other half not before (dk, sk)
          const int h = (lo + hi) >> 1;
          const uint32_t sh = src[h];
          if (item_before(a.geo[sh].depth, sh, dk, sk))
            lo = h + 1;
          else
            hi = h;
        }
        dst[b0 + own + (lo - (left ? mid : b0))] = sk;
      }
      __syncthreads();
      uint32_t* t = src;
      src = dst;
      dst = t;
    }
    if (src != base) {
      for (int k = threadIdx.x; k < L; k += blockDim.x) base[k] = src[k];
    }
    __syncthreads();
  }
}

__global__ void item_counts_kernel(NarrowArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_items) return;
  a.item_count[i] = a.counts[a.item_slot_sorted[i]];
}

// K3n: visible items in depth order write their tile pairs (key = global tile
// id) and record their pair offset under their slot (VF finalize). A warp takes
// 32 consecutive items, whose pairs form one contiguous range, and writes that
// range lane-strided (coalesced): each pair finds its item by a binary search
// over the 32 item offsets and its tile from the item's rectangle.
__global__ void __launch_bounds__(256) emit_tiles_kernel(EmitArgs a, NarrowArgs n) {
  __shared__ int32_t s_off[8][33];
  __shared__ int32_t s_tb[8][32], s_tx[8][32], s_x0[8][32], s_y0[8][32], s_w[8][32];
  __shared__ uint32_t s_g[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i0 = ((int64_t)blockIdx.x * 8 + warp) * 32;
  if (i0 >= n.n_items) return;
  const int nv = (int)min((int64_t)32, n.n_items - i0);
  const int64_t i = i0 + lane;
  if (lane < nv) {
    const uint32_t slot = n.item_slot_sorted[i];
    const int v = (int)(slot / (uint32_t)a.N);
    const DevCam& c = a.cams[v];
    const uint2 tr = a.trect[slot];
    const int tx0 = tr.x & 0xFFFF, tx1 = tr.x >> 16, ty0 = tr.y & 0xFFFF;
    const int32_t o = n.item_offset[i];
    n.slot_offset[slot] = o;
    s_off[warp][lane] = o;
    s_tb[warp][lane] = (int32_t)(c.tile_base - n.chunk_tile_base[v]);
    s_tx[warp][lane] = c.tiles_x;
    s_x0[warp][lane] = tx0;
    s_y0[warp][lane] = ty0;
    s_w[warp][lane] = tx1 - tx0 + 1;
    s_g[warp][lane] = slot - (uint32_t)v * (uint32_t)a.N;
    if (lane == nv - 1) s_off[warp][32] = o + n.item_count[i];
  }
  __syncwarp();
  const int32_t start = s_off[warp][0], end = s_off[warp][32];
  for (int32_t p = start + lane; p < end; p += 32) {
    int j = 0;
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (j + step < nv && s_off[warp][j + step] <= p) j += step;
    const int k = p - s_off[warp][j];
    const int w = s_w[warp][j];
    const int dy = k / w, dx = k - dy * w;
    n.keys32[p] = (uint32_t)(s_tb[warp][j] + (s_y0[warp][j] + dy) * s_tx[warp][j] + s_x0[warp][j] + dx);
    const uint32_t g = s_g[warp][j];
    if (a.pair_gid) {
      a.vals[p] = (uint32_t)p;
      a.pair_gid[p] = g;
    } else {
      a.vals[p] = g;
    }
  }
}

// K5n: tile ranges of the tile-sorted pairs [lo, hi) of one chunk of views
// (keys = tile id - tile_base).
__global__ void ranges32_kernel(const uint32_t* keys32, int64_t lo, int64_t hi, int64_t tile_base,
                                uint2* ranges) {
  const int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= hi) return;
  const uint32_t t = keys32[i];
  if (i == lo || keys32[i - 1] != t) ranges[tile_base + t].x = (uint32_t)i;
  if (i == hi - 1 || keys32[i + 1] != t) ranges[tile_base + t].y = (uint32_t)(i + 1);
}

// Pair offset of the first item of every view (lower bound of the view's key
// prefix in the depth-sorted items); out[V] = K.
__global__ void view_pair_starts_kernel(NarrowArgs a, int V, int64_t* out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v > V) return;
  if (v == V) {
    out[V] = a.item_offset[a.n_items];
    return;
  }
  const uint32_t key = (uint32_t)v << (32 - a.view_bits);
  int64_t lo = 0, hi = a.n_items;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (a.item_key[mid] < key) lo = mid + 1; else hi = mid;
  }
  out[v] = a.item_offset[lo];
}

// Reference-form 64-bit keys (tile << 32 | fp32 depth) of the sorted pairs, for
// gavis_debug_binning.
__global__ void wide_keys_kernel(const uint2* ranges, int64_t total_tiles, const uint32_t* vals,
                                 const uint32_t* pair_gid, const DevCam* cams, int V, int64_t N,
                                 const GeoRec* geo, uint64_t* keys) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= total_tiles) return;
  int v = 0;
  while (v + 1 < V && cams[v + 1].tile_base <= t) ++v;
  const uint2 r = ranges[t];
  for (uint32_t i = r.x; i < r.y; ++i) {
    const uint32_t g = pair_gid ? pair_gid[vals[i]] : vals[i];
    const float df = __double2float_rz(geo[(int64_t)v * N + g].depth);
    keys[i] = ((uint64_t)t << 32) | (uint64_t)__float_as_uint(df);
  }
}

template <int DEG>
__global__ void query_kernel(QueryArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  constexpr int NB = (DEG + 1) * (DEG + 1);
  const int64_t g = a.idx[i];
  double out = 0.0;
  if (!(a.virt && a.virt[g]) && a.num_views > 0) {
    double row[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) row[k] = a.gamma[g * NB + k];
    out = query_row<DEG>(row, a.num_views, a.dirs[3 * i], a.dirs[3 * i + 1], a.dirs[3 * i + 2]);
  }
  a.out[i] = out;
}

__global__ void query_rt_kernel(QueryArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int nb = (a.degree + 1) * (a.degree + 1);
  const int64_t g = a.idx[i];
  double out = 0.0;
  if (!(a.virt && a.virt[g]) && a.num_views > 0)
    out = query_row_rt(a.gamma + g * nb, a.degree, a.num_views, a.dirs[3 * i], a.dirs[3 * i + 1],
                       a.dirs[3 * i + 2]);
  a.out[i] = out;
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

void launch_preprocess(const PreprocessArgs& a, cudaStream_t s) {
  if (a.scene.n == 0 || a.V == 0) return;
  const unsigned grid = blocks_for(a.scene.n, kPreThreads);
  const int qd = a.query_mode == kQueryField ? a.degree : -1;
  switch (qd) {
    case -1: preprocess_kernel<-1><<<grid, kPreThreads, 0, s>>>(a); break;
    case 0: preprocess_kernel<0><<<grid, kPreThreads, 0, s>>>(a); break;
    case 1: preprocess_kernel<1><<<grid, kPreThreads, 0, s>>>(a); break;
    case 2: preprocess_kernel<2><<<grid, kPreThreads, 0, s>>>(a); break;
    case 3: preprocess_kernel<3><<<grid, kPreThreads, 0, s>>>(a); break;
    case 4: preprocess_kernel<4><<<grid, kPreThreads, 0, s>>>(a); break;
    default: preprocess_kernel<kDegRT><<<grid, kPreThreads, 0, s>>>(a); break;
  }
}

void launch_emit_keys(const EmitArgs& a, cudaStream_t s) {
  const int64_t n = (int64_t)a.V * a.N;
  if (n == 0) return;
  emit_keys_kernel<<<blocks_for(n, 256), 256, 0, s>>>(a);
}

void launch_depth_order(const NarrowArgs& a, cudaStream_t s) {
  if (a.n_items == 0) return;
  cudaMemsetAsync(a.n_long, 0, sizeof(uint32_t), s);
  depth_order_kernel<<<blocks_for(a.n_items, 256), 256, 0, s>>>(a);
  depth_order_long_kernel<<<148, 256, 0, s>>>(a);
  item_counts_kernel<<<blocks_for(a.n_items, 256), 256, 0, s>>>(a);
}

void launch_emit_tiles(const EmitArgs& a, const NarrowArgs& n, cudaStream_t s) {
  if (n.n_items > 0) emit_tiles_kernel<<<blocks_for(n.n_items, 256), 256, 0, s>>>(a, n);  // 32 items per warp
}

void launch_ranges32(const uint32_t* keys32, int64_t lo, int64_t hi, int64_t tile_base, uint2* ranges,
                     cudaStream_t s) {
  if (hi > lo)
    ranges32_kernel<<<blocks_for(hi - lo, 256), 256, 0, s>>>(keys32, lo, hi, tile_base, ranges);
}

void launch_view_pair_starts(const NarrowArgs& a, int V, int64_t* out, cudaStream_t s) {
  view_pair_starts_kernel<<<blocks_for(V + 1, 64), 64, 0, s>>>(a, V, out);
}

void launch_wide_keys(const uint2* ranges, int64_t total_tiles, const uint32_t* vals,
                      const uint32_t* pair_gid, const DevCam* cams, int V, int64_t N, const GeoRec* geo,
                      uint64_t* keys, cudaStream_t s) {
  if (total_tiles > 0)
    wide_keys_kernel<<<blocks_for(total_tiles, 128), 128, 0, s>>>(ranges, total_tiles, vals, pair_gid,
                                                                 cams, V, N, geo, keys);
}

void launch_ranges(const RangesArgs& a, cudaStream_t s) {
  if (a.K == 0) return;
  ranges_kernel<<<blocks_for(a.K, 256), 256, 0, s>>>(a);
}

// Scene upload: host SoA (positions [N][3], opacities [N], scales [N][3],
// colours [N][3][nb], is_virtual [N]) staged raw in device memory -> the device
// layout (float4 pos|opacity, float4 scale, colour rows padded to nbp, 0/1 mask).
__global__ void pack_scene_kernel(PackSceneArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  a.pos_op[i] = make_float4(a.pos[3 * i], a.pos[3 * i + 1], a.pos[3 * i + 2], a.op[i]);
  a.scale4[i] = make_float4(a.scale[3 * i], a.scale[3 * i + 1], a.scale[3 * i + 2], 0.f);
  a.virt_out[i] = a.virt ? (a.virt[i] ? 1 : 0) : 0;
  if (a.colors) {
    float* dst = a.colors_out + i * a.cstride;
    const float* src = a.colors + i * 3 * a.nb;
    for (int k = 0; k < a.cstride; ++k) {
      const int ch = k / a.nbp, m = k - ch * a.nbp;
      dst[k] = (ch < 3 && m < a.nb) ? src[ch * a.nb + m] : 0.f;
    }
  }
}

void launch_pack_scene(const PackSceneArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  pack_scene_kernel<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a);
}

void launch_query(const QueryArgs& a, cudaStream_t s) {
  if (a.n == 0) return;
  const unsigned grid = blocks_for(a.n, 128);
  switch (a.degree) {
    case 0: query_kernel<0><<<grid, 128, 0, s>>>(a); break;
    case 1: query_kernel<1><<<grid, 128, 0, s>>>(a); break;
    case 2: query_kernel<2><<<grid, 128, 0, s>>>(a); break;
    case 3: query_kernel<3><<<grid, 128, 0, s>>>(a); break;
    case 4: query_kernel<4><<<grid, 128, 0, s>>>(a); break;
    default: query_rt_kernel<<<grid, 128, 0, s>>>(a); break;
  }
}

}  // namespace gavis
