/*
 * gavis_oracle.c -- CPU ORACLE (test infrastructure only; see gavis_oracle.h).
 *
 * Double-precision restatement of the GAVIS reference hot path. Each function
 * cites the reference lines it follows (R/ = /root/reference/proj/). Build with
 * -O3 -ffp-contract=off (the reference is CMake Release, no -march, so no FMA
 * contraction: R/CMakeLists.txt:8-10). Eigen's fixed-size 3x3 products are
 * restated as left-to-right sums over the inner index.
 */
#include "gavis_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

#define K_PI 3.14159265358979323846
#define K_Y00 0.28209479177387814
#define K_GAUSS_ENTROPY 4.256815599614018
#define MAX_SH 21 * 21

/* parallel_for, R/include/gavis/parallel.hpp:35-60: static block partition
 * [n*w/T, n*(w+1)/T) over T worker threads. */
typedef void (*body_fn)(int i, void* ctx);
typedef struct {
  body_fn body;
  void* ctx;
  int begin, end;
} pf_task;

static void* pf_worker(void* arg) {
  pf_task* t = (pf_task*)arg;
  for (int i = t->begin; i < t->end; ++i) t->body(i, t->ctx);
  return NULL;
}

static void parallel_for(int n, int threads, body_fn body, void* ctx) {
  if (threads < 1) threads = 1;
  if (threads > n) threads = n > 0 ? n : 1;
  if (threads <= 1 || n <= 1) {
    for (int i = 0; i < n; ++i) body(i, ctx);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  pf_task* tasks = (pf_task*)malloc(sizeof(pf_task) * (size_t)threads);
  for (int w = 0; w < threads; ++w) {
    tasks[w].body = body;
    tasks[w].ctx = ctx;
    tasks[w].begin = (int)((long long)n * w / threads);
    tasks[w].end = (int)((long long)n * (w + 1) / threads);
    pthread_create(&th[w], NULL, pf_worker, &tasks[w]);
  }
  for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
  free(th);
  free(tasks);
}

/* ---------------------------------------------------------------- sh.hpp */

/* eval_real_sh_block, R/include/gavis/sh.hpp:38-79 */
void gor_eval_sh(int degree, const double* d, double* out) {
  const double x = d[0], y = d[1], z = d[2];
  const double s = sqrt(x * x + y * y);
  const double cphi = s > 1e-14 ? x / s : 1.0;
  const double sphi = s > 1e-14 ? y / s : 0.0;
  const double kSqrt2 = 1.4142135623730951;
  double pmm = K_Y00;
  double cm = 1.0, sm = 0.0;
  for (int m = 0; m <= degree; ++m) {
    if (m > 0) {
      pmm *= s * sqrt((2.0 * m + 1.0) / (2.0 * m));
      double cnext = cm * cphi - sm * sphi;
      sm = sm * cphi + cm * sphi;
      cm = cnext;
    }
    double plm = pmm, plm_prev = 0.0;
    for (int l = m; l <= degree; ++l) {
      if (l > m) {
        double next;
        if (l == m + 1) {
          next = z * sqrt(2.0 * m + 3.0) * pmm;
        } else {
          double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
          double b = sqrt(((double)(l - 1) * (l - 1) - (double)m * m) /
                          (4.0 * (double)(l - 1) * (l - 1) - 1.0));
          next = a * (z * plm - b * plm_prev);
        }
        plm_prev = plm;
        plm = next;
      }
      if (m == 0) {
        out[l * l + l] = plm;
      } else {
        out[l * l + l + m] = kSqrt2 * plm * cm;
        out[l * l + l - m] = kSqrt2 * plm * sm;
      }
    }
  }
}

/* bessel_i, sh.hpp:93-119 */
double gor_bessel_i(int l, double x) {
  if (x == 0.0) return l == 0 ? 1.0 : 0.0;
  if (l == 0) return sinh(x) / x;
  if (l == 1) return (x * cosh(x) - sinh(x)) / (x * x);
  if (x >= 2.0 * l + 2.0) {
    double prev = sinh(x) / x;
    double cur = (x * cosh(x) - sinh(x)) / (x * x);
    for (int k = 1; k < l; ++k) {
      double next = prev - (2.0 * k + 1.0) / x * cur;
      prev = cur;
      cur = next;
    }
    return cur;
  }
  double term = pow(x, l);
  for (int k = 3; k <= 2 * l + 1; k += 2) term /= k;
  double sum = term;
  const double x2h = 0.5 * x * x;
  for (int k = 1; k < 400; ++k) {
    term *= x2h / (k * (2.0 * l + 2.0 * k + 1.0));
    sum += term;
    if (term <= sum * 1e-17) break;
  }
  return sum;
}

/* VmfParams(kappa) sh.hpp:121-129 + vmf_degree_scales sh.hpp:140-147 */
void gor_vmf_scales(double kappa, int degree, double* scales) {
  const double zeta = exp(-kappa);
  for (int l = 0; l <= degree; ++l) scales[l] = 4.0 * K_PI * zeta * gor_bessel_i(l, kappa);
}

/* ------------------------------------------------------------- model.hpp */

typedef struct {
  double fx, fy, cx, cy, limx, limy;
} cam_derived;

/* CameraView::focal_x/focal_y/cx/cy model.hpp:75-78; limits raster.hpp:60-61 */
static cam_derived derive(const gor_camera* c) {
  cam_derived d;
  d.fx = 0.5 * c->width / tan(0.5 * c->fov_h);
  d.fy = 0.5 * c->height / tan(0.5 * c->fov_v);
  d.cx = 0.5 * c->width;
  d.cy = 0.5 * c->height;
  d.limx = 1.3 * tan(0.5 * c->fov_h);
  d.limy = 1.3 * tan(0.5 * c->fov_v);
  return d;
}

#define RM(c, r, k) ((c)->rotation[(r) * 3 + (k)])

/* CameraView::pixel_ray model.hpp:83-86 */
static void pixel_ray(const gor_camera* c, const cam_derived* cd, double px, double py,
                      double* out) {
  double dc[3] = {(px - cd->cx) / cd->fx, (py - cd->cy) / cd->fy, 1.0};
  double r[3];
  for (int i = 0; i < 3; ++i) r[i] = RM(c, i, 0) * dc[0] + RM(c, i, 1) * dc[1] + RM(c, i, 2) * dc[2];
  double n2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
  if (n2 > 0.0) {
    double n = sqrt(n2);
    for (int i = 0; i < 3; ++i) out[i] = r[i] / n;
  } else {
    for (int i = 0; i < 3; ++i) out[i] = r[i];
  }
}

/* GaussianParticle::covariance model.hpp:42-45 (Eigen Quaternion::toRotationMatrix) */
static void covariance(const gor_scene* s, int64_t i, double sig[9]) {
  const double w = s->rotations[4 * i], x = s->rotations[4 * i + 1];
  const double y = s->rotations[4 * i + 2], z = s->rotations[4 * i + 3];
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  double R[9] = {1.0 - (tyy + tzz), txy - twz, txz + twy,
                 txy + twz, 1.0 - (txx + tzz), tyz - twx,
                 txz - twy, tyz + twx, 1.0 - (txx + tyy)};
  double sc[3] = {s->scales[3 * i], s->scales[3 * i + 1], s->scales[3 * i + 2]};
  double m[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m[r * 3 + c] = R[r * 3 + c] * sc[c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      sig[r * 3 + c] = m[r * 3 + 0] * m[c * 3 + 0] + m[r * 3 + 1] * m[c * 3 + 1] +
                       m[r * 3 + 2] * m[c * 3 + 2];
}

/* ------------------------------------------------------------ raster.hpp */

/* project_particle raster.hpp:51-93 */
static int project_particle_d(const gor_scene* s, int64_t i, const gor_camera* cam,
                              const cam_derived* cd, double dilation, gor_splat* out) {
  double p[3] = {s->positions[3 * i], s->positions[3 * i + 1], s->positions[3 * i + 2]};
  double dd[3] = {p[0] - cam->position[0], p[1] - cam->position[1], p[2] - cam->position[2]};
  double t[3];
  for (int k = 0; k < 3; ++k)
    t[k] = RM(cam, 0, k) * dd[0] + RM(cam, 1, k) * dd[1] + RM(cam, 2, k) * dd[2];
  if (t[2] < cam->near_plane) return 0;
  const double fx = cd->fx, fy = cd->fy;
  const double inv_z = 1.0 / t[2];
  double mx = cd->cx + fx * t[0] * inv_z;
  double my = cd->cy + fy * t[1] * inv_z;
  double ux = t[0] * inv_z, uy = t[1] * inv_z;
  ux = ux < -cd->limx ? -cd->limx : (cd->limx < ux ? cd->limx : ux);
  uy = uy < -cd->limy ? -cd->limy : (cd->limy < uy ? cd->limy : uy);
  const double jx = ux * t[2];
  const double jy = uy * t[2];
  double sig[9];
  covariance(s, i, sig);
  /* w2c = R^T: W(r,k) = R(k,r); cov_cam = (W Sigma) W^T */
  double A[9], C[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      A[r * 3 + c] = RM(cam, 0, r) * sig[0 * 3 + c] + RM(cam, 1, r) * sig[1 * 3 + c] +
                     RM(cam, 2, r) * sig[2 * 3 + c];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c)
      C[r * 3 + c] = A[r * 3 + 0] * RM(cam, 0, c) + A[r * 3 + 1] * RM(cam, 1, c) +
                     A[r * 3 + 2] * RM(cam, 2, c);
  double J[6] = {fx * inv_z, 0.0, -fx * jx * inv_z * inv_z,
                 0.0, fy * inv_z, -fy * jy * inv_z * inv_z};
  double B[6], c2[4];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 3; ++c)
      B[r * 3 + c] = J[r * 3 + 0] * C[0 * 3 + c] + J[r * 3 + 1] * C[1 * 3 + c] +
                     J[r * 3 + 2] * C[2 * 3 + c];
  for (int r = 0; r < 2; ++r)
    for (int c = 0; c < 2; ++c)
      c2[r * 2 + c] = B[r * 3 + 0] * J[c * 3 + 0] + B[r * 3 + 1] * J[c * 3 + 1] +
                      B[r * 3 + 2] * J[c * 3 + 2];
  c2[0] += dilation * dilation;
  c2[3] += dilation * dilation;
  double det = c2[0] * c2[3] - c2[1] * c2[2];
  if (det <= 0.0) return 0;
  double mid = 0.5 * (c2[0] + c2[3]);
  double disc = mid * mid - det;
  double lam_max = mid + sqrt(disc > 0.0 ? disc : 0.0);
  double radius = 3.0 * sqrt(lam_max);
  if (mx < -radius || mx > cam->width + radius || my < -radius || my > cam->height + radius)
    return 0;
  double inv_det = 1.0 / det;
  out->particle_index = (int32_t)i;
  out->mean_x = mx;
  out->mean_y = my;
  out->conic_a = c2[3] * inv_det;
  out->conic_b = -c2[1] * inv_det;
  out->conic_c = c2[0] * inv_det;
  out->depth = t[2];
  out->radius = radius;
  out->opacity = s->opacities[i];
  return 1;
}

int gor_project_particle(const gor_scene* s, int64_t i, const gor_camera* cam, double dilation,
                         gor_splat* out) {
  cam_derived cd = derive(cam);
  return project_particle_d(s, i, cam, &cd, dilation, out);
}

/* splat_covers raster.hpp:97-99 */
static inline int splat_covers(const gor_splat* s, double px, double py) {
  return fabs(px - s->mean_x) <= s->radius && fabs(py - s->mean_y) <= s->radius;
}

/* splat_alpha raster.hpp:101-108 */
static inline double splat_alpha(const gor_splat* s, double px, double py, double amax) {
  double dx = px - s->mean_x;
  double dy = py - s->mean_y;
  double q = s->conic_a * dx * dx + 2.0 * s->conic_b * dx * dy + s->conic_c * dy * dy;
  double a = s->opacity * exp(-0.5 * q);
  return a > amax ? amax : a;
}

static int cmp_splat(const void* a, const void* b) {
  const gor_splat* x = (const gor_splat*)a;
  const gor_splat* y = (const gor_splat*)b;
  if (x->depth != y->depth) return x->depth < y->depth ? -1 : 1;
  return x->particle_index < y->particle_index ? -1 : (x->particle_index > y->particle_index);
}

/* project_scene raster.hpp:114-130 */
int64_t gor_project_scene(const gor_scene* s, const gor_camera* cam, double dilation,
                          gor_splat* out) {
  cam_derived cd = derive(cam);
  int64_t n = 0;
  for (int64_t i = 0; i < s->num_particles; ++i)
    if (project_particle_d(s, i, cam, &cd, dilation, &out[n])) ++n;
  qsort(out, (size_t)n, sizeof(gor_splat), cmp_splat);
  return n;
}

/* covered_pixel_range raster.hpp:138-141 */
void gor_covered_pixel_range(double m, double r, int n, int* lo, int* hi) {
  int a = (int)ceil(m - r - 0.5);
  int b = (int)floor(m + r - 0.5);
  *lo = a > 0 ? a : 0;
  *hi = b < n - 1 ? b : n - 1;
}

/* splat_binning raster.hpp:145-164, as CSR over tiles */
int64_t gor_splat_binning(const gor_splat* splats, int64_t n, int width, int height,
                          int tile_size, int64_t* tile_offsets, int32_t* entries) {
  const int tx_n = (width + tile_size - 1) / tile_size;
  const int ty_n = (height + tile_size - 1) / tile_size;
  const int64_t tiles = (int64_t)tx_n * ty_n;
  int64_t* cnt = (int64_t*)calloc((size_t)tiles + 1, sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) {
    int x0, x1, y0, y1;
    gor_covered_pixel_range(splats[k].mean_x, splats[k].radius, width, &x0, &x1);
    gor_covered_pixel_range(splats[k].mean_y, splats[k].radius, height, &y0, &y1);
    if (x0 > x1 || y0 > y1) continue;
    for (int ty = y0 / tile_size; ty <= y1 / tile_size; ++ty)
      for (int tx = x0 / tile_size; tx <= x1 / tile_size; ++tx) cnt[(int64_t)ty * tx_n + tx + 1]++;
  }
  for (int64_t t = 0; t < tiles; ++t) cnt[t + 1] += cnt[t];
  int64_t total = cnt[tiles];
  if (tile_offsets) memcpy(tile_offsets, cnt, sizeof(int64_t) * (size_t)(tiles + 1));
  if (entries) {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)tiles);
    memcpy(fill, cnt, sizeof(int64_t) * (size_t)tiles);
    for (int64_t k = 0; k < n; ++k) {
      int x0, x1, y0, y1;
      gor_covered_pixel_range(splats[k].mean_x, splats[k].radius, width, &x0, &x1);
      gor_covered_pixel_range(splats[k].mean_y, splats[k].radius, height, &y0, &y1);
      if (x0 > x1 || y0 > y1) continue;
      for (int ty = y0 / tile_size; ty <= y1 / tile_size; ++ty)
        for (int tx = x0 / tile_size; tx <= x1 / tile_size; ++tx)
          entries[fill[(int64_t)ty * tx_n + tx]++] = (int32_t)k;
    }
    free(fill);
  }
  free(cnt);
  return total;
}

typedef struct {
  gor_splat* splats;
  int64_t n;
  int tx_n, ty_n;
  int64_t* off;
  int32_t* ent;
} binned_view;

static binned_view bin_view(const gor_scene* s, const gor_camera* cam, const gor_raster* rc) {
  binned_view b;
  b.splats = (gor_splat*)malloc(sizeof(gor_splat) * (size_t)(s->num_particles + 1));
  b.n = gor_project_scene(s, cam, rc->dilation, b.splats);
  b.tx_n = (cam->width + rc->tile_size - 1) / rc->tile_size;
  b.ty_n = (cam->height + rc->tile_size - 1) / rc->tile_size;
  int64_t tiles = (int64_t)b.tx_n * b.ty_n;
  b.off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(tiles + 1));
  int64_t total = gor_splat_binning(b.splats, b.n, cam->width, cam->height, rc->tile_size, b.off, NULL);
  b.ent = (int32_t*)malloc(sizeof(int32_t) * (size_t)(total + 1));
  gor_splat_binning(b.splats, b.n, cam->width, cam->height, rc->tile_size, b.off, b.ent);
  return b;
}

static void free_view(binned_view* b) {
  free(b->splats);
  free(b->off);
  free(b->ent);
}

static inline double clamp01(double v) { return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v); }

/* rasterize raster.hpp:175-231 (tile loop run sequentially; results are
 * thread-count independent by construction in the reference) */
void gor_rasterize(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                   double* rgb, double* depth, double* trans, int32_t* contrib) {
  binned_view b = bin_view(s, cam, rc);
  cam_derived cd = derive(cam);
  const int W = cam->width, H = cam->height, ts = rc->tile_size;
  const int degree = s->color_degree;
  const int nb = (degree + 1) * (degree + 1);
  double basis[MAX_SH];
  for (int64_t p = 0; p < (int64_t)W * H; ++p) {
    rgb[3 * p] = rgb[3 * p + 1] = rgb[3 * p + 2] = 0.0;
    if (depth) depth[p] = 0.0;
    if (trans) trans[p] = 1.0;
    if (contrib) contrib[p] = 0;
  }
  for (int tile = 0; tile < b.tx_n * b.ty_n; ++tile) {
    int tx = tile % b.tx_n, ty = tile / b.tx_n;
    int px0 = tx * ts, px1 = px0 + ts < W ? px0 + ts : W;
    int py0 = ty * ts, py1 = py0 + ts < H ? py0 + ts : H;
    for (int py = py0; py < py1; ++py) {
      for (int px = px0; px < px1; ++px) {
        const double cxp = px + 0.5, cyp = py + 0.5;
        double ray[3];
        pixel_ray(cam, &cd, cxp, cyp, ray);
        gor_eval_sh(degree, ray, basis);
        double t_cur = 1.0, acc[3] = {0.0, 0.0, 0.0}, depth_acc = 0.0;
        int32_t nc = 0;
        for (int64_t e = b.off[tile]; e < b.off[tile + 1]; ++e) {
          const gor_splat* sp = &b.splats[b.ent[e]];
          if (!splat_covers(sp, cxp, cyp)) continue;
          ++nc;
          double a = splat_alpha(sp, cxp, cyp, rc->alpha_clamp_max);
          double w = a * t_cur;
          if (w > 0.0) {
            const double* col = s->colors + (int64_t)sp->particle_index * 3 * nb;
            for (int k = 0; k < 3; ++k) {
              double c = 0.0;
              for (int i = 0; i < nb; ++i) c += col[k * nb + i] * basis[i];
              acc[k] += w * clamp01(c);
            }
            depth_acc += w * sp->depth;
          }
          t_cur *= 1.0 - a;
          if (t_cur < rc->transmittance_cutoff) break;
        }
        int64_t pix = (int64_t)py * W + px;
        for (int k = 0; k < 3; ++k) rgb[pix * 3 + k] = acc[k];
        if (depth) depth[pix] = depth_acc;
        if (trans) trans[pix] = t_cur;
        if (contrib) contrib[pix] = nc;
      }
    }
  }
  free_view(&b);
}

/* brute_force_rasterize, R/tests/test_raster.cpp:50-85 (tile-free reference) */
void gor_rasterize_brute(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                         double* rgb, double* depth, double* trans) {
  gor_splat* sp = (gor_splat*)malloc(sizeof(gor_splat) * (size_t)(s->num_particles + 1));
  int64_t n = gor_project_scene(s, cam, rc->dilation, sp);
  cam_derived cd = derive(cam);
  const int degree = s->color_degree;
  const int nb = (degree + 1) * (degree + 1);
  double basis[MAX_SH];
  for (int py = 0; py < cam->height; ++py) {
    for (int px = 0; px < cam->width; ++px) {
      const double cxp = px + 0.5, cyp = py + 0.5;
      double ray[3];
      pixel_ray(cam, &cd, cxp, cyp, ray);
      gor_eval_sh(degree, ray, basis);
      double t_cur = 1.0, acc[3] = {0, 0, 0}, depth_acc = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        if (!splat_covers(&sp[k], cxp, cyp)) continue;
        double a = splat_alpha(&sp[k], cxp, cyp, rc->alpha_clamp_max);
        double w = a * t_cur;
        if (w > 0.0) {
          const double* col = s->colors + (int64_t)sp[k].particle_index * 3 * nb;
          for (int c = 0; c < 3; ++c) {
            double v = 0.0;
            for (int i = 0; i < nb; ++i) v += col[c * nb + i] * basis[i];
            acc[c] += w * clamp01(v);
          }
          depth_acc += w * sp[k].depth;
        }
        t_cur *= 1.0 - a;
        if (t_cur < rc->transmittance_cutoff) break;
      }
      int64_t pix = (int64_t)py * cam->width + px;
      for (int c = 0; c < 3; ++c) rgb[pix * 3 + c] = acc[c];
      depth[pix] = depth_acc;
      trans[pix] = t_cur;
    }
  }
  free(sp);
}

/* single_view_visibility raster.hpp:237-290 */
void gor_single_view_visibility(const gor_scene* s, const gor_camera* cam,
                                const gor_raster* rc, double* vis, int64_t* touch_out,
                                int32_t* contrib) {
  binned_view b = bin_view(s, cam, rc);
  const int W = cam->width, H = cam->height, ts = rc->tile_size;
  const int64_t total = b.off[(int64_t)b.tx_n * b.ty_n];
  double* tvis = (double*)calloc((size_t)total + 1, sizeof(double));
  long long* tcnt = (long long*)calloc((size_t)total + 1, sizeof(long long));
  if (contrib)
    for (int64_t p = 0; p < (int64_t)W * H; ++p) contrib[p] = 0;
  for (int tile = 0; tile < b.tx_n * b.ty_n; ++tile) {
    int64_t e0 = b.off[tile], e1 = b.off[tile + 1];
    if (e0 == e1) continue;
    int tx = tile % b.tx_n, ty = tile / b.tx_n;
    int px0 = tx * ts, px1 = px0 + ts < W ? px0 + ts : W;
    int py0 = ty * ts, py1 = py0 + ts < H ? py0 + ts : H;
    for (int py = py0; py < py1; ++py) {
      for (int px = px0; px < px1; ++px) {
        const double cxp = px + 0.5, cyp = py + 0.5;
        double t_cur = 1.0;
        int32_t nc = 0;
        for (int64_t e = e0; e < e1; ++e) {
          const gor_splat* sp = &b.splats[b.ent[e]];
          if (!splat_covers(sp, cxp, cyp)) continue;
          ++nc;
          tvis[e] += t_cur;
          tcnt[e] += 1;
          double a = splat_alpha(sp, cxp, cyp, rc->alpha_clamp_max);
          t_cur *= 1.0 - a;
          if (t_cur < rc->transmittance_cutoff) break;
        }
        if (contrib) contrib[(int64_t)py * W + px] = nc;
      }
    }
  }
  const int64_t N = s->num_particles;
  double* vsum = (double*)calloc((size_t)N + 1, sizeof(double));
  long long* touch = (long long*)calloc((size_t)N + 1, sizeof(long long));
  for (int64_t tile = 0; tile < (int64_t)b.tx_n * b.ty_n; ++tile) {
    for (int64_t e = b.off[tile]; e < b.off[tile + 1]; ++e) {
      int particle = b.splats[b.ent[e]].particle_index;
      vsum[particle] += tvis[e];
      touch[particle] += tcnt[e];
    }
  }
  for (int64_t i = 0; i < N; ++i) {
    vis[i] = touch[i] > 0 ? vsum[i] / (double)touch[i] : 0.0;
    if (touch_out) touch_out[i] = touch[i];
  }
  free(tvis);
  free(tcnt);
  free(vsum);
  free(touch);
  free_view(&b);
}

/* ------------------------------------------------------------ vfield.hpp */

/* accumulate_view vfield.hpp:38-63 */
void gor_accumulate_view(double* gamma, int degree, double kappa, const gor_scene* s,
                         const gor_camera* view, const double* vis) {
  double scales[21];
  gor_vmf_scales(kappa, degree, scales);
  const int nb = (degree + 1) * (degree + 1);
  double basis[MAX_SH];
  for (int64_t i = 0; i < s->num_particles; ++i) {
    if ((s->is_virtual && s->is_virtual[i]) || vis[i] <= 0.0) continue;
    double d[3] = {s->positions[3 * i] - view->position[0],
                   s->positions[3 * i + 1] - view->position[1],
                   s->positions[3 * i + 2] - view->position[2]};
    double norm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (norm < 1e-12) continue;
    d[0] /= norm;
    d[1] /= norm;
    d[2] /= norm;
    gor_eval_sh(degree, d, basis);
    double* row = gamma + i * nb;
    for (int l = 0; l <= degree; ++l) {
      double scale = vis[i] * scales[l];
      for (int m = -l; m <= l; ++m) {
        int idx = l * l + l + m;
        row[idx] += scale * basis[idx];
      }
    }
  }
}

typedef struct {
  const gor_scene* s;
  const gor_camera* views;
  const gor_raster* rc;
  double* per_view;
  int64_t N;
} cf_ctx;

static void cf_body(int v, void* p) {
  cf_ctx* c = (cf_ctx*)p;
  gor_single_view_visibility(c->s, &c->views[v], c->rc, c->per_view + (int64_t)v * (c->N + 1),
                             NULL, NULL);
}

/* construct_field vfield.hpp:68-92: views rendered in parallel, folded in order */
void gor_construct_field(const gor_scene* s, const gor_camera* views, int n_views,
                         double kappa, int degree, const gor_raster* rc, int threads,
                         double* gamma) {
  const int nb = (degree + 1) * (degree + 1);
  const int64_t N = s->num_particles;
  memset(gamma, 0, sizeof(double) * (size_t)(N * nb));
  double* per_view = (double*)malloc(sizeof(double) * (size_t)(N + 1) * (size_t)n_views);
  cf_ctx cx = {s, views, rc, per_view, N};
  parallel_for(n_views, threads, cf_body, &cx);
  for (int v = 0; v < n_views; ++v)
    gor_accumulate_view(gamma, degree, kappa, s, &views[v], per_view + (int64_t)v * (N + 1));
  free(per_view);
}

/* query_visibility vfield.hpp:96-112 */
double gor_query_visibility(const double* row, int degree, int num_views, int is_virtual,
                            const double* d) {
  if (is_virtual) return 0.0;
  if (num_views <= 0) return 0.0;
  double basis[MAX_SH];
  gor_eval_sh(degree, d, basis);
  const int nb = (degree + 1) * (degree + 1);
  double vt = 0.0;
  for (int i = 0; i < nb; ++i) vt += row[i] * basis[i];
  const double p = (double)num_views;
  if (vt < 0.0) vt = 0.0;
  if (vt > p) vt = p;
  double v = 1.0 - pow(1.0 - vt / p, p);
  return clamp01(v);
}

/* query_view vfield.hpp:121-134 */
int64_t gor_query_view(const double* gamma, int degree, int num_views, const gor_scene* s,
                       const gor_camera* cam, double dilation, int32_t* idx, double* vis) {
  cam_derived cd = derive(cam);
  const int nb = (degree + 1) * (degree + 1);
  int64_t n = 0;
  for (int64_t i = 0; i < s->num_particles; ++i) {
    gor_splat sp;
    if (!project_particle_d(s, i, cam, &cd, dilation, &sp)) continue;
    double d[3] = {s->positions[3 * i] - cam->position[0],
                   s->positions[3 * i + 1] - cam->position[1],
                   s->positions[3 * i + 2] - cam->position[2]};
    double n2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    if (n2 > 0.0) {
      double nn = sqrt(n2);
      d[0] /= nn;
      d[1] /= nn;
      d[2] /= nn;
    }
    idx[n] = (int32_t)i;
    vis[n] = gor_query_visibility(gamma + i * nb, degree, num_views,
                                  s->is_virtual ? s->is_virtual[i] : 0, d);
    ++n;
  }
  return n;
}

/* ------------------------------------------------------- uncertainty.hpp */

/* compensated_alpha uncertainty.hpp:55-59 */
static inline double compensated_alpha(double alpha, double v, const gor_unc* uc, double amax) {
  double a = (v + uc->beta * (1.0 - v)) * alpha + uc->prior_opacity * (1.0 - uc->beta) * (1.0 - v);
  return a < 0.0 ? 0.0 : (amax < a ? amax : a);
}

/* detail::logdet_spd uncertainty.hpp:108-113 (unblocked Cholesky of a 3x3) */
static double logdet_spd3(const double* m) {
  double L[9] = {0};
  for (int k = 0; k < 3; ++k) {
    double sq = 0.0;
    for (int j = 0; j < k; ++j) sq += L[k * 3 + j] * L[k * 3 + j];
    double x = k > 0 ? m[k * 3 + k] - sq : m[k * 3 + k];
    L[k * 3 + k] = sqrt(x);
    for (int r = k + 1; r < 3; ++r) {
      double dot = 0.0;
      for (int j = 0; j < k; ++j) dot += L[r * 3 + j] * L[k * 3 + j];
      double y = k > 0 ? m[r * 3 + k] - dot : m[r * 3 + k];
      L[r * 3 + k] = y / L[k * 3 + k];
    }
  }
  return 2.0 * (log(L[0]) + log(L[4]) + log(L[8]));
}

/* UncertaintyConfig::coeff_variances (uncertainty.hpp:38): [N][3][(Lv+1)^2] */
static const double* g_coeff_var = NULL;
static int g_coeff_var_degree = -1;

void gor_set_coeff_variances(const double* var, int degree) {
  g_coeff_var = var;
  g_coeff_var_degree = degree;
}

/* sh_variance_propagation uncertainty.hpp:63-83; returns 0 if a q <= 0 */
static int propagated_half_logdet(const double* var, int degree, const double* d, double* hl) {
  double basis[MAX_SH];
  gor_eval_sh(degree, d, basis);
  const int n = (degree + 1) * (degree + 1);
  double q[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < n; ++i) {
    double y2 = basis[i] * basis[i];
    for (int k = 0; k < 3; ++k) q[k] += y2 * var[k * n + i];
  }
  if (!(q[0] > 0.0 && q[1] > 0.0 && q[2] > 0.0)) return 0;
  *hl = 0.5 * (log(q[0]) + log(q[1]) + log(q[2]));
  return 1;
}

/* render_entropy_core uncertainty.hpp:124-238; variance_provider 1 uses the
 * coefficient variances set by gor_set_coeff_variances (:149-163). */
void gor_render_entropy_core(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                             const gor_unc* uc, const double* vis_by_particle, double* entropy,
                             double* w0_out, double* depth_out, int32_t* contrib) {
  binned_view b = bin_view(s, cam, rc);
  const double hl_const = 3.0 * log(uc->color_sigma);
  const double hl_q0 = 0.5 * logdet_spd3(uc->prior_cov);
  double* hl_of = NULL; /* per sorted splat */
  if (uc->variance_provider == 1) {
    hl_of = (double*)malloc(sizeof(double) * (size_t)(b.n + 1));
    const int nbv = (g_coeff_var_degree + 1) * (g_coeff_var_degree + 1);
    for (int64_t k = 0; k < b.n; ++k) {
      const int64_t i = b.splats[k].particle_index;
      double d[3] = {s->positions[3 * i] - cam->position[0], s->positions[3 * i + 1] - cam->position[1],
                     s->positions[3 * i + 2] - cam->position[2]};
      double n2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
      if (n2 > 0.0) {
        double nn = sqrt(n2);
        d[0] /= nn;
        d[1] /= nn;
        d[2] /= nn;
      }
      if (!propagated_half_logdet(g_coeff_var + i * 3 * nbv, g_coeff_var_degree, d, &hl_of[k]))
        hl_of[k] = NAN;
    }
  }
  const int W = cam->width, H = cam->height, ts = rc->tile_size;
  for (int tile = 0; tile < b.tx_n * b.ty_n; ++tile) {
    int tx = tile % b.tx_n, ty = tile / b.tx_n;
    int px0 = tx * ts, px1 = px0 + ts < W ? px0 + ts : W;
    int py0 = ty * ts, py1 = py0 + ts < H ? py0 + ts : H;
    for (int py = py0; py < py1; ++py) {
      for (int px = px0; px < px1; ++px) {
        const double cxp = px + 0.5, cyp = py + 0.5;
        int64_t pix = (int64_t)py * W + px;
        double t_cur = 1.0, h = 0.0, w0 = 0.0, depth_acc = 0.0;
        int32_t nc = 0;
        for (int64_t e = b.off[tile]; e < b.off[tile + 1]; ++e) {
          const gor_splat* sp = &b.splats[b.ent[e]];
          if (!splat_covers(sp, cxp, cyp)) continue;
          ++nc;
          double a = splat_alpha(sp, cxp, cyp, rc->alpha_clamp_max);
          double v = vis_by_particle[sp->particle_index];
          double astar = compensated_alpha(a, v, uc, rc->alpha_clamp_max);
          double w = astar * t_cur;
          double seen = w * v;
          const double hl_qc = hl_of ? hl_of[b.ent[e]] : hl_const;
          if (seen > 0.0) h += seen * (-log(seen) + hl_qc + K_GAUSS_ENTROPY);
          w0 += w * (1.0 - v);
          depth_acc += w * sp->depth;
          t_cur *= 1.0 - astar;
          if (t_cur < rc->transmittance_cutoff) break;
        }
        if (w0 > 0.0) h += w0 * (-log(w0) + hl_q0 + K_GAUSS_ENTROPY);
        entropy[pix] = h;
        if (w0_out) w0_out[pix] = w0;
        if (depth_out) depth_out[pix] = depth_acc;
        if (contrib) contrib[pix] = nc;
      }
    }
  }
  free(hl_of);
  free_view(&b);
}

/* render_entropy_core's per-pixel mixtures (uncertainty.hpp:90-102, :185-230):
 * for every composited entry with w* > 0, in list order, the component
 * {w*, v, clamp(SH colour at the pixel ray), diag Q_c}; per pixel the prior
 * weight w0, the residual T* and the entropy. offsets[P+1] always; comps only
 * when non-NULL (capacity >= offsets[P] checked by the caller). */
void gor_render_mixtures(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                         const gor_unc* uc, const double* vis_by_particle, int64_t* offsets,
                         gor_mixture_component* comps, double* prior, double* resid,
                         double* entropy) {
  binned_view b = bin_view(s, cam, rc);
  cam_derived cd = derive(cam);
  const double hl_const = 3.0 * log(uc->color_sigma);
  const double hl_q0 = 0.5 * logdet_spd3(uc->prior_cov);
  const double var_const = uc->color_sigma * uc->color_sigma;
  const int degree = s->color_degree;
  const int nb = (degree + 1) * (degree + 1);
  const int W = cam->width, H = cam->height, ts = rc->tile_size;
  const int nbv = (g_coeff_var_degree + 1) * (g_coeff_var_degree + 1);
  int64_t* count = (int64_t*)calloc((size_t)W * H + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      offsets[0] = 0;
      for (int64_t p = 0; p < (int64_t)W * H; ++p) offsets[p + 1] = offsets[p] + count[p];
      if (!comps) break;
    }
    for (int tile = 0; tile < b.tx_n * b.ty_n; ++tile) {
      int tx = tile % b.tx_n, ty = tile / b.tx_n;
      int px0 = tx * ts, px1 = px0 + ts < W ? px0 + ts : W;
      int py0 = ty * ts, py1 = py0 + ts < H ? py0 + ts : H;
      for (int py = py0; py < py1; ++py) {
        for (int px = px0; px < px1; ++px) {
          const double cxp = px + 0.5, cyp = py + 0.5;
          const int64_t pix = (int64_t)py * W + px;
          double ray[3], basis[MAX_SH];
          pixel_ray(cam, &cd, cxp, cyp, ray);
          gor_eval_sh(degree, ray, basis);
          double t_cur = 1.0, h = 0.0, w0 = 0.0;
          int64_t k = 0;
          for (int64_t e = b.off[tile]; e < b.off[tile + 1]; ++e) {
            const gor_splat* sp = &b.splats[b.ent[e]];
            if (!splat_covers(sp, cxp, cyp)) continue;
            const int64_t i = sp->particle_index;
            double a = splat_alpha(sp, cxp, cyp, rc->alpha_clamp_max);
            double v = vis_by_particle[i];
            double astar = compensated_alpha(a, v, uc, rc->alpha_clamp_max);
            double w = astar * t_cur;
            double seen = w * v;
            double qd[3] = {var_const, var_const, var_const}, hl_qc = hl_const;
            if (uc->variance_provider == 1) {
              double d[3] = {s->positions[3 * i] - cam->position[0],
                             s->positions[3 * i + 1] - cam->position[1],
                             s->positions[3 * i + 2] - cam->position[2]};
              double n2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
              if (n2 > 0.0) {
                double nn = sqrt(n2);
                d[0] /= nn;
                d[1] /= nn;
                d[2] /= nn;
              }
              double bv[MAX_SH];
              gor_eval_sh(g_coeff_var_degree, d, bv);
              qd[0] = qd[1] = qd[2] = 0.0;
              for (int j = 0; j < nbv; ++j)
                for (int c = 0; c < 3; ++c) qd[c] += bv[j] * bv[j] * g_coeff_var[i * 3 * nbv + c * nbv + j];
              hl_qc = 0.5 * (log(qd[0]) + log(qd[1]) + log(qd[2]));
            }
            if (seen > 0.0) h += seen * (-log(seen) + hl_qc + K_GAUSS_ENTROPY);
            w0 += w * (1.0 - v);
            if (w > 0.0) {
              if (pass == 0) {
                ++count[pix];
              } else {
                gor_mixture_component* m = &comps[offsets[pix] + k];
                m->weight = w;
                m->vis = v;
                const double* col = s->colors + i * 3 * nb;
                for (int c = 0; c < 3; ++c) {
                  double acc = 0.0;
                  for (int j = 0; j < nb; ++j) acc += col[c * nb + j] * basis[j];
                  m->mean[c] = clamp01(acc);
                  m->var[c] = qd[c];
                }
              }
              ++k;
            }
            t_cur *= 1.0 - astar;
            if (t_cur < rc->transmittance_cutoff) break;
          }
          if (w0 > 0.0) h += w0 * (-log(w0) + hl_q0 + K_GAUSS_ENTROPY);
          if (pass == 0) {
            if (prior) prior[pix] = w0;
            if (resid) resid[pix] = t_cur;
            if (entropy) entropy[pix] = h;
          }
        }
      }
    }
  }
  free(count);
  free_view(&b);
}

/* render_entropy uncertainty.hpp:242-260: per-splat visibility from the field */
void gor_splat_visibility(const double* gamma, int degree, int num_views, const gor_scene* s,
                          const gor_camera* cam, double dilation, double* vis) {
  cam_derived cd = derive(cam);
  const int nb = (degree + 1) * (degree + 1);
  for (int64_t i = 0; i < s->num_particles; ++i) {
    vis[i] = 0.0;
    gor_splat sp;
    if (!project_particle_d(s, i, cam, &cd, dilation, &sp)) continue;
    double d[3] = {s->positions[3 * i] - cam->position[0],
                   s->positions[3 * i + 1] - cam->position[1],
                   s->positions[3 * i + 2] - cam->position[2]};
    double norm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (norm < 1e-12) continue;
    double dn[3] = {d[0] / norm, d[1] / norm, d[2] / norm};
    vis[i] = gor_query_visibility(gamma + i * nb, degree, num_views,
                                  s->is_virtual ? s->is_virtual[i] : 0, dn);
  }
}

void gor_render_entropy(const gor_scene* s, const double* gamma, int degree, int num_views,
                        const gor_camera* cam, const gor_raster* rc, const gor_unc* uc,
                        double* entropy, double* w0, double* depth, int32_t* contrib) {
  double* vis = (double*)malloc(sizeof(double) * (size_t)(s->num_particles + 1));
  gor_splat_visibility(gamma, degree, num_views, s, cam, rc->dilation, vis);
  gor_render_entropy_core(s, cam, rc, uc, vis, entropy, w0, depth, contrib);
  free(vis);
}

/* image_entropy uncertainty.hpp:264-278 (correlation none) */
double gor_image_entropy(const double* entropy, int64_t n) {
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) sum += entropy[i];
  return sum;
}

/* image_entropy with the correlation hook uncertainty.hpp:273-277 */
double gor_image_entropy_hook(const double* entropy, const double* depth, int64_t n, double lambda) {
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double h = entropy[i];
    sum += h - h * exp(-depth[i] / lambda);
  }
  return sum;
}

/* ------------------------------------------------------------ planner.hpp */

typedef struct {
  const gor_scene* s;
  const double* gamma;
  int degree, num_views;
  const gor_camera* cams;
  const gor_raster* rc;
  const gor_unc* uc;
  int with_rgb;
  double* scores;
} nbv_ctx;

static void nbv_body(int c, void* p) {
  nbv_ctx* x = (nbv_ctx*)p;
  const int64_t P = (int64_t)x->cams[c].width * x->cams[c].height;
  double* ent = (double*)malloc(sizeof(double) * (size_t)P);
  if (x->with_rgb) {
    double* rgb = (double*)malloc(sizeof(double) * (size_t)P * 3);
    gor_rasterize(x->s, &x->cams[c], x->rc, rgb, NULL, NULL, NULL);
    free(rgb);
  }
  if (x->uc->correlation == 1) { /* planner.hpp:124-130: depth for the hook */
    double* dep = (double*)malloc(sizeof(double) * (size_t)P);
    gor_render_entropy(x->s, x->gamma, x->degree, x->num_views, &x->cams[c], x->rc, x->uc, ent,
                       NULL, dep, NULL);
    x->scores[c] = gor_image_entropy_hook(ent, dep, P, x->uc->correlation_lambda);
    free(dep);
  } else {
    gor_render_entropy(x->s, x->gamma, x->degree, x->num_views, &x->cams[c], x->rc, x->uc, ent,
                       NULL, NULL, NULL);
    x->scores[c] = gor_image_entropy(ent, P);
  }
  free(ent);
}

/* select_nbv planner.hpp:117-137 */
int gor_select_nbv(const gor_scene* s, const double* gamma, int degree, int num_views,
                   const gor_camera* cams, int n_cams, const gor_raster* rc,
                   const gor_unc* uc, int threads, int with_rgb, double* scores) {
  nbv_ctx cx = {s, gamma, degree, num_views, cams, rc, uc, with_rgb, scores};
  parallel_for(n_cams, threads, nbv_body, &cx);
  int best = 0;
  for (int c = 1; c < n_cams; ++c)
    if (scores[c] > scores[best]) best = c;
  return best;
}

/* ------------------------------------------------------------- oracle.hpp */

/* ------------------------------------------------ rng.hpp + density control */

static uint64_t mix64_(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

/* derive_seed rng.hpp:26-28 */
uint64_t gor_derive_seed(uint64_t seed, uint64_t stream) {
  return mix64_(seed ^ mix64_(stream + 0x632be59bd9b4e019ull));
}

/* SplitMix64::next_double rng.hpp:35-45 */
static double sm_next_double(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z = z ^ (z >> 31);
  return (double)(z >> 11) * 0x1.0p-53;
}

/* density_control vfield.hpp:149-199 */
int64_t gor_density_control(const gor_scene* s, const double* bmin, const double* bmax,
                            const gor_camera* views, int n_views, double rho, double eta,
                            double eps_v, uint64_t seed, const gor_raster* rc, int threads,
                            int round_f32, int64_t* kept_ids, double* unseen_out) {
  const double ext[3] = {bmax[0] - bmin[0], bmax[1] - bmin[1], bmax[2] - bmin[2]};
  const double volume = ext[0] * ext[1] * ext[2];
  const int64_t n_virtual = (int64_t)floor(rho * volume);
  const int64_t n_real = s->num_particles;
  const int64_t n = n_real + n_virtual;
  const int nb = (s->color_degree + 1) * (s->color_degree + 1);
  double sc = cbrt(3.0 * (1.0 + eta) / (4.0 * K_PI * rho));
  if (round_f32) sc = (double)(float)sc;
  double* pos = (double*)malloc(sizeof(double) * 3 * (size_t)(n + 1));
  double* rot = (double*)malloc(sizeof(double) * 4 * (size_t)(n + 1));
  double* scl = (double*)malloc(sizeof(double) * 3 * (size_t)(n + 1));
  double* op = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  double* col = (double*)calloc((size_t)(3 * nb * (n + 1)), sizeof(double));
  uint8_t* virt = (uint8_t*)calloc((size_t)(n + 1), 1);
  memcpy(pos, s->positions, sizeof(double) * 3 * (size_t)n_real);
  memcpy(rot, s->rotations, sizeof(double) * 4 * (size_t)n_real);
  memcpy(scl, s->scales, sizeof(double) * 3 * (size_t)n_real);
  memcpy(op, s->opacities, sizeof(double) * (size_t)n_real);
  memcpy(col, s->colors, sizeof(double) * 3 * nb * (size_t)n_real);
  if (s->is_virtual) memcpy(virt, s->is_virtual, (size_t)n_real);
  for (int64_t k = 0; k < n_virtual; ++k) {
    uint64_t st = gor_derive_seed(seed, (uint64_t)k);
    const double ux = sm_next_double(&st), uy = sm_next_double(&st), uz = sm_next_double(&st);
    const double u[3] = {ux, uy, uz};
    const int64_t i = n_real + k;
    for (int d = 0; d < 3; ++d) {
      double p = bmin[d] + ext[d] * u[d];
      pos[3 * i + d] = round_f32 ? (double)(float)p : p;
      scl[3 * i + d] = sc;
    }
    rot[4 * i] = 1.0;
    rot[4 * i + 1] = rot[4 * i + 2] = rot[4 * i + 3] = 0.0;
    op[i] = 0.0;
    virt[i] = 1;
  }
  gor_scene probe = {n, s->color_degree, 0, pos, rot, scl, op, col, virt};
  double* unseen = (double*)malloc(sizeof(double) * (size_t)(n_virtual + 1));
  for (int64_t k = 0; k < n_virtual; ++k) unseen[k] = 1.0;
  double* b = (double*)malloc(sizeof(double) * (size_t)(n + 1));
  (void)threads;
  for (int v = 0; v < n_views; ++v) {
    gor_single_view_visibility(&probe, &views[v], rc, b, NULL, NULL);
    for (int64_t k = 0; k < n_virtual; ++k) unseen[k] *= 1.0 - b[n_real + k];
  }
  int64_t kept = 0;
  for (int64_t k = 0; k < n_virtual; ++k) {
    if (unseen_out) unseen_out[k] = unseen[k];
    double vtilde = 1.0 - unseen[k];
    if (vtilde > eps_v) continue;
    if (kept_ids) kept_ids[kept] = k;
    ++kept;
  }
  free(pos);
  free(rot);
  free(scl);
  free(op);
  free(col);
  free(virt);
  free(unseen);
  free(b);
  return kept;
}

/* raymarch_transmittance oracle.hpp:70-103 */
double gor_raymarch_transmittance(const gor_scene* s, const double* origin,
                                  const double* target, double step, int64_t exclude,
                                  double alpha_clamp_max) {
  double span[3] = {target[0] - origin[0], target[1] - origin[1], target[2] - origin[2]};
  double length = sqrt(span[0] * span[0] + span[1] * span[1] + span[2] * span[2]);
  if (length < 1e-12) return 1.0;
  double dir[3] = {span[0] / length, span[1] / length, span[2] / length};
  int n_steps = (int)ceil(length / step);
  if (n_steps < 1) n_steps = 1;
  double tr = 1.0;
  for (int64_t i = 0; i < s->num_particles; ++i) {
    if (i == exclude) continue;
    double op = s->opacities[i];
    if (op <= 0.0) continue;
    double c[9], inv[9];
    covariance(s, i, c);
    double det = c[0] * (c[4] * c[8] - c[5] * c[7]) - c[1] * (c[3] * c[8] - c[5] * c[6]) +
                 c[2] * (c[3] * c[7] - c[4] * c[6]);
    inv[0] = (c[4] * c[8] - c[5] * c[7]) / det;
    inv[1] = (c[2] * c[7] - c[1] * c[8]) / det;
    inv[2] = (c[1] * c[5] - c[2] * c[4]) / det;
    inv[3] = (c[5] * c[6] - c[3] * c[8]) / det;
    inv[4] = (c[0] * c[8] - c[2] * c[6]) / det;
    inv[5] = (c[2] * c[3] - c[0] * c[5]) / det;
    inv[6] = (c[3] * c[7] - c[4] * c[6]) / det;
    inv[7] = (c[1] * c[6] - c[0] * c[7]) / det;
    inv[8] = (c[0] * c[4] - c[1] * c[3]) / det;
    double e[3] = {origin[0] - s->positions[3 * i], origin[1] - s->positions[3 * i + 1],
                   origin[2] - s->positions[3 * i + 2]};
    double pd[3], pe[3];
    for (int r = 0; r < 3; ++r) {
      pd[r] = inv[r * 3] * dir[0] + inv[r * 3 + 1] * dir[1] + inv[r * 3 + 2] * dir[2];
      pe[r] = inv[r * 3] * e[0] + inv[r * 3 + 1] * e[1] + inv[r * 3 + 2] * e[2];
    }
    double qa = dir[0] * pd[0] + dir[1] * pd[1] + dir[2] * pd[2];
    double qb = 2.0 * (dir[0] * pe[0] + dir[1] * pe[1] + dir[2] * pe[2]);
    double qc = e[0] * pe[0] + e[1] * pe[1] + e[2] * pe[2];
    double q_min = INFINITY;
    for (int k = 0; k < n_steps; ++k) {
      double t = (k + 0.5) * length / n_steps;
      double q = (qa * t + qb) * t + qc;
      if (q < q_min) q_min = q;
    }
    double alpha = op * exp(-0.5 * q_min);
    if (alpha > alpha_clamp_max) alpha = alpha_clamp_max;
    tr *= 1.0 - alpha;
  }
  return tr;
}

/* ------------------------------------------------------------------------- */
/* planner.hpp:45-107 (sample_candidates) and :141-184 (vis_coverage).       */
/* Eigen fixed-size kernels written out: 3x3 determinant / cofactor inverse   */
/* (Eigen LU module), Quaternion::normalized + toRotationMatrix.              */

typedef struct {
  uint64_t state;
} gor_sm64;

static uint64_t sm64_next(gor_sm64* g) { /* rng.hpp:34-40 */
  g->state += 0x9e3779b97f4a7c15ull;
  return mix64_(g->state - 0x9e3779b97f4a7c15ull);
}
static double sm64_double(gor_sm64* g) { return (double)(sm64_next(g) >> 11) * 0x1.0p-53; }
static double sm64_uniform(gor_sm64* g, double lo, double hi) { return lo + (hi - lo) * sm64_double(g); }

static double v3_norm(const double* a) { return sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); }
static void v3_cross(const double* a, const double* b, double* o) {
  o[0] = a[1] * b[2] - a[2] * b[1];
  o[1] = a[2] * b[0] - a[0] * b[2];
  o[2] = a[0] * b[1] - a[1] * b[0];
}

/* make_lookat, model.hpp:107-128, up = (0,0,1). Returns 0 on coincident points. */
static int lookat_(const double* pos, const double* target, gor_camera* cam) {
  double f[3] = {target[0] - pos[0], target[1] - pos[1], target[2] - pos[2]};
  if (!(v3_norm(f) > 1e-12)) return 0;
  double n = v3_norm(f);
  for (int i = 0; i < 3; ++i) f[i] /= n;
  const double up[3] = {0.0, 0.0, 1.0}, ex[3] = {1.0, 0.0, 0.0};
  double r[3], d[3];
  v3_cross(f, up, r);
  if (v3_norm(r) < 1e-9) v3_cross(f, ex, r);
  n = v3_norm(r);
  for (int i = 0; i < 3; ++i) r[i] /= n;
  v3_cross(f, r, d);
  for (int i = 0; i < 3; ++i) {
    cam->rotation[i * 3 + 0] = r[i];
    cam->rotation[i * 3 + 1] = d[i];
    cam->rotation[i * 3 + 2] = f[i];
  }
  return 1;
}

/* rect: corner[3], edge_u[3], edge_v[3], opaque flag (layout of gor_rect). */
static double rect_dist_(const gor_rect* rc, const double* p) { /* planner.hpp:45-52 */
  double w[3], uu = 0, vv = 0, wu, wv;
  for (int i = 0; i < 3; ++i) w[i] = p[i] - rc->corner[i];
  uu = rc->edge_u[0] * rc->edge_u[0] + rc->edge_u[1] * rc->edge_u[1] + rc->edge_u[2] * rc->edge_u[2];
  vv = rc->edge_v[0] * rc->edge_v[0] + rc->edge_v[1] * rc->edge_v[1] + rc->edge_v[2] * rc->edge_v[2];
  wu = w[0] * rc->edge_u[0] + w[1] * rc->edge_u[1] + w[2] * rc->edge_u[2];
  wv = w[0] * rc->edge_v[0] + w[1] * rc->edge_v[1] + w[2] * rc->edge_v[2];
  double u = 0.0, v = 0.0;
  if (uu > 0.0) { u = wu / uu; u = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u); }
  if (vv > 0.0) { v = wv / vv; v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }
  double q[3];
  for (int i = 0; i < 3; ++i) q[i] = (rc->corner[i] + u * rc->edge_u[i]) + v * rc->edge_v[i] - p[i];
  return v3_norm(q);
}

int gor_sample_candidates(const double* bmin, const double* bmax, const gor_rect* rects,
                          int n_rects, const gor_planner* pc, uint64_t step_seed, gor_camera* out) {
  const double ext[3] = {bmax[0] - bmin[0], bmax[1] - bmin[1], bmax[2] - bmin[2]};
  if (!(ext[0] * ext[1] * ext[2] > 0.0) || pc->num_candidates < 1) return -1;
  gor_sm64 g = {gor_derive_seed(step_seed, 0xca4d1d)};
  long long budget = 100LL * pc->num_candidates, attempts = 0;
  int n = 0;
  while (n < pc->num_candidates) {
    if (attempts++ >= budget) return -2;
    double p[3];
    /* planner.hpp:70-72 draws the three coordinates as the arguments of one Vec3
     * constructor call, whose evaluation order C++ leaves unspecified; GCC (the
     * reference's Linux build, and oracle/_ref here) evaluates them right to
     * left: z, then y, then x. */
    for (int i = 2; i >= 0; --i) p[i] = sm64_uniform(&g, bmin[i], bmax[i]);
    const double yaw = sm64_uniform(&g, 0.0, 2.0 * K_PI);
    const double u1 = sm64_double(&g), u2 = sm64_double(&g), u3 = sm64_double(&g);
    const double qa = sqrt(1.0 - u1), qb = sqrt(u1);
    /* Quat(w, x, y, z) = (a sin 2pi u2, a cos 2pi u2, b sin 2pi u3, b cos 2pi u3) */
    const double qw = qa * sin(2.0 * K_PI * u2), qx = qa * cos(2.0 * K_PI * u2);
    const double qy = qb * sin(2.0 * K_PI * u3), qz = qb * cos(2.0 * K_PI * u3);
    if (pc->mode == 1) p[2] = pc->se2_height;
    int hit = 0;
    for (int r = 0; r < n_rects && !hit; ++r)
      if (rects[r].opaque && rect_dist_(&rects[r], p) < pc->clearance) hit = 1;
    if (hit) continue;
    gor_camera cam;
    memset(&cam, 0, sizeof(cam));
    if (pc->mode == 1) {
      const double t[3] = {p[0] + cos(yaw), p[1] + sin(yaw), p[2] + 0.0};
      if (!lookat_(p, t, &cam)) return -3;
    } else if (pc->look_inward) {
      double t[3] = {0.5 * (bmin[0] + bmax[0]), 0.5 * (bmin[1] + bmax[1]), 0.5 * (bmin[2] + bmax[2])};
      const double dd[3] = {t[0] - p[0], t[1] - p[1], t[2] - p[2]};
      if (v3_norm(dd) < 1e-9) t[0] += 1e-3;
      if (!lookat_(p, t, &cam)) return -3;
    } else {
      /* Eigen stores (x, y, z, w); SSE2 squaredNorm = (x^2 + z^2) + (y^2 + w^2) */
      const double nq = sqrt((qx * qx + qz * qz) + (qy * qy + qw * qw));
      const double w = qw / nq, x = qx / nq, y = qy / nq, z = qz / nq;
      const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
      double* R = cam.rotation;
      R[0] = 1 - (ty * y + tz * z);
      R[1] = ty * x - tz * w;
      R[2] = tz * x + ty * w;
      R[3] = ty * x + tz * w;
      R[4] = 1 - (tx * x + tz * z);
      R[5] = tz * y - tx * w;
      R[6] = tz * x - ty * w;
      R[7] = tz * y + tx * w;
      R[8] = 1 - (tx * x + ty * y);
    }
    for (int i = 0; i < 3; ++i) cam.position[i] = p[i];
    cam.width = pc->cam_width;
    cam.height = pc->cam_height;
    cam.fov_h = pc->fov_h;
    cam.fov_v = pc->fov_v;
    cam.near_plane = pc->cam_near;
    out[n++] = cam;
  }
  return n;
}

/* intersect_rect, model.hpp:157-175 */
static int isect_(const gor_rect* rc, const double* o, const double* dir, double* t_out) {
  double m[9] = {rc->edge_u[0], rc->edge_v[0], -dir[0], rc->edge_u[1], rc->edge_v[1], -dir[1],
                 rc->edge_u[2], rc->edge_v[2], -dir[2]};
#define M_(r, c) m[(r) * 3 + (c)]
  const double det = M_(0, 0) * (M_(1, 1) * M_(2, 2) - M_(1, 2) * M_(2, 1)) -
                     M_(0, 1) * (M_(1, 0) * M_(2, 2) - M_(1, 2) * M_(2, 0)) +
                     M_(0, 2) * (M_(1, 0) * M_(2, 1) - M_(1, 1) * M_(2, 0));
  if (fabs(det) < 1e-14) return 0;
  /* cofactor C(i,j) = M(i1,j1) M(i2,j2) - M(i1,j2) M(i2,j1), i1 = i+1, i2 = i+2 mod 3 */
  double C[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
      C[i * 3 + j] = M_(i1, j1) * M_(i2, j2) - M_(i1, j2) * M_(i2, j1);
    }
  const double d2 = (C[0] * M_(0, 0) + C[3] * M_(1, 0)) + C[6] * M_(2, 0);
#undef M_
  const double inv_det = 1.0 / d2;
  /* inverse = adjugate / det: inv(i, j) = C(j, i) * inv_det */
  const double w[3] = {o[0] - rc->corner[0], o[1] - rc->corner[1], o[2] - rc->corner[2]};
  double sol[3];
  for (int i = 0; i < 3; ++i)
    sol[i] = (C[0 * 3 + i] * inv_det) * w[0] + (C[1 * 3 + i] * inv_det) * w[1] + (C[2 * 3 + i] * inv_det) * w[2];
  if (sol[0] < 0.0 || sol[0] > 1.0 || sol[1] < 0.0 || sol[1] > 1.0) return 0;
  *t_out = sol[2];
  return 1;
}

/* CameraView::project, model.hpp:90-97 */
static int project_(const gor_camera* c, const double* p) {
  const double d[3] = {p[0] - c->position[0], p[1] - c->position[1], p[2] - c->position[2]};
  double cc[3];
  for (int i = 0; i < 3; ++i)
    cc[i] = c->rotation[0 * 3 + i] * d[0] + c->rotation[1 * 3 + i] * d[1] + c->rotation[2 * 3 + i] * d[2];
  if (cc[2] < c->near_plane) return 0;
  const double fx = 0.5 * c->width / tan(0.5 * c->fov_h), fy = 0.5 * c->height / tan(0.5 * c->fov_v);
  const double px = 0.5 * c->width + fx * cc[0] / cc[2], py = 0.5 * c->height + fy * cc[1] / cc[2];
  return px >= 0.0 && px <= c->width && py >= 0.0 && py <= c->height;
}

double gor_vis_coverage(const gor_rect* rects, int n_rects, double density, const gor_camera* views,
                        int n_views) {
  double total = 0.0, vis = 0.0;
  for (int r = 0; r < n_rects; ++r) {
    const gor_rect* rc = &rects[r];
    double cr[3];
    v3_cross(rc->edge_u, rc->edge_v, cr);
    const double area = v3_norm(cr);
    total += area;
    if (n_views == 0) continue;
    const double ps = sqrt(density);
    int nu = (int)lround(v3_norm(rc->edge_u) * ps), nv = (int)lround(v3_norm(rc->edge_v) * ps);
    if (nu < 1) nu = 1;
    if (nv < 1) nv = 1;
    long long seen = 0;
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nv; ++j) {
        const double u = (i + 0.5) / nu, v = (j + 0.5) / nv;
        double p[3];
        for (int k = 0; k < 3; ++k) p[k] = (rc->corner[k] + u * rc->edge_u[k]) + v * rc->edge_v[k];
        for (int k = 0; k < n_views; ++k) {
          const gor_camera* c = &views[k];
          if (!project_(c, p)) continue;
          const double seg[3] = {p[0] - c->position[0], p[1] - c->position[1], p[2] - c->position[2]};
          int blocked = 0;
          for (int q = 0; q < n_rects && !blocked; ++q) {
            double t;
            if (!rects[q].opaque || q == r) continue;
            if (isect_(&rects[q], c->position, seg, &t) && t > 1e-9 && t < 1.0 - 1e-9) blocked = 1;
          }
          if (!blocked) {
            ++seen;
            break;
          }
        }
      }
    vis += area * (double)seen / ((double)nu * nv);
  }
  return total > 0.0 ? vis / total : 0.0;
}
