/*
 * gavis_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C, double-precision restatement of the GAVIS reference hot path
 * (/root/reference/proj/include/gavis/{sh,model,raster,vfield,uncertainty,planner}.hpp).
 * It exists to CHECK the CUDA product, never to stand in for it: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.
 *
 * Parity pin: every known-answer test the reference's own suite holds for this
 * path is re-run against this oracle in tests/test_oracle_kats.py.
 *
 * Camera/config layouts match include/gavis_b200.h. The scene is taken in
 * double (the reference's own type, common.hpp:14-18); parity runs feed it the
 * exact fp32 values the CUDA path consumes.
 */
#ifndef GAVIS_ORACLE_H
#define GAVIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  double rotation[9]; /* row-major 3x3 camera-to-world; columns = right, down, forward */
  double position[3];
  int32_t width, height;
  double fov_h, fov_v, near_plane;
} gor_camera;

typedef struct {
  int32_t tile_size;
  int32_t _pad;
  double transmittance_cutoff, dilation, alpha_clamp_max;
} gor_raster;

typedef struct {
  double beta, prior_opacity, color_sigma;
  double prior_cov[9];
  int32_t variance_provider, correlation;
  double correlation_lambda;
} gor_unc;

typedef struct {
  int64_t num_particles;
  int32_t color_degree, _pad;
  const double* positions; /* [N*3] */
  const double* rotations; /* [N*4] w,x,y,z */
  const double* scales;    /* [N*3] */
  const double* opacities; /* [N]   */
  const double* colors;    /* [N*3*(Lc+1)^2] per particle, channel-major */
  const uint8_t* is_virtual; /* [N] or NULL */
} gor_scene;

/* ImageSpaceSplat (raster.hpp:37-44) */
typedef struct {
  int32_t particle_index, _pad;
  double mean_x, mean_y, conic_a, conic_b, conic_c, depth, radius, opacity;
} gor_splat;

/* sh.hpp */
void gor_eval_sh(int degree, const double* d, double* out);
double gor_bessel_i(int l, double x);
void gor_vmf_scales(double kappa, int degree, double* scales);

/* raster.hpp */
int gor_project_particle(const gor_scene* s, int64_t i, const gor_camera* cam, double dilation,
                         gor_splat* out);
int64_t gor_project_scene(const gor_scene* s, const gor_camera* cam, double dilation,
                          gor_splat* out);
void gor_covered_pixel_range(double m, double r, int n, int* lo, int* hi);
/* CSR tile lists; entries index the sorted splat array. Pass entries=NULL to size. */
int64_t gor_splat_binning(const gor_splat* splats, int64_t n, int width, int height,
                          int tile_size, int64_t* tile_offsets, int32_t* entries);
void gor_rasterize(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                   double* rgb, double* depth, double* trans, int32_t* contrib);
void gor_rasterize_brute(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                         double* rgb, double* depth, double* trans);
void gor_single_view_visibility(const gor_scene* s, const gor_camera* cam,
                                const gor_raster* rc, double* vis, int64_t* touch,
                                int32_t* contrib);

/* vfield.hpp */
void gor_accumulate_view(double* gamma, int degree, double kappa, const gor_scene* s,
                         const gor_camera* view, const double* vis);
void gor_construct_field(const gor_scene* s, const gor_camera* views, int n_views,
                         double kappa, int degree, const gor_raster* rc, int threads,
                         double* gamma);
double gor_query_visibility(const double* row, int degree, int num_views, int is_virtual,
                            const double* d);
int64_t gor_query_view(const double* gamma, int degree, int num_views, const gor_scene* s,
                       const gor_camera* cam, double dilation, int32_t* idx, double* vis);

/* uncertainty.hpp: vis_by_particle indexed by particle id */
/* PixelMixtureComponent (uncertainty.hpp:90-95) */
typedef struct {
  double weight, vis, mean[3], var[3];
} gor_mixture_component;
void gor_render_mixtures(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                         const gor_unc* uc, const double* vis_by_particle, int64_t* offsets,
                         gor_mixture_component* comps, double* prior, double* resid,
                         double* entropy);
void gor_render_entropy_core(const gor_scene* s, const gor_camera* cam, const gor_raster* rc,
                             const gor_unc* uc, const double* vis_by_particle, double* entropy,
                             double* w0, double* depth, int32_t* contrib);
void gor_splat_visibility(const double* gamma, int degree, int num_views, const gor_scene* s,
                          const gor_camera* cam, double dilation, double* vis_by_particle);
void gor_render_entropy(const gor_scene* s, const double* gamma, int degree, int num_views,
                        const gor_camera* cam, const gor_raster* rc, const gor_unc* uc,
                        double* entropy, double* w0, double* depth, int32_t* contrib);
double gor_image_entropy(const double* entropy, int64_t n);
double gor_image_entropy_hook(const double* entropy, const double* depth, int64_t n, double lambda);
/* coefficient variances [N][3][(Lv+1)^2] for variance_provider 1 (NULL to clear) */
void gor_set_coeff_variances(const double* var, int degree);

/* planner.hpp: returns best index; with_rgb additionally runs rasterize per
 * candidate (the fused GPU render's RGB work) and discards it. */
int gor_select_nbv(const gor_scene* s, const double* gamma, int degree, int num_views,
                   const gor_camera* cams, int n_cams, const gor_raster* rc,
                   const gor_unc* uc, int threads, int with_rgb, double* scores);

/* density_control vfield.hpp:157-199: appends the retained virtual probes to a
 * copy of the scene arrays. Writes kept probe ids (k) into kept_ids (capacity
 * n_virtual = floor(rho * volume)) and returns their count. round_f32 != 0 rounds
 * the probe position/scale to fp32 first (what the device stores). */
int64_t gor_density_control(const gor_scene* s, const double* bounds_min, const double* bounds_max,
                            const gor_camera* views, int n_views, double rho, double eta,
                            double eps_v, uint64_t seed, const gor_raster* rc, int threads,
                            int round_f32, int64_t* kept_ids, double* unseen_out);
uint64_t gor_derive_seed(uint64_t seed, uint64_t stream);

/* planner.hpp:24-42 PlannerConfig / model.hpp:141-150 OccluderRect (layouts of
 * gavis_planner_config / gavis_occluder_rect). */
typedef struct {
  int32_t mode, num_candidates;
  double se2_height;
  int32_t steps, look_inward;
  uint64_t seed;
  double clearance;
  int32_t cam_width, cam_height;
  double fov_h, fov_v, cam_near;
} gor_planner;

typedef struct {
  double corner[3], edge_u[3], edge_v[3];
  int32_t opaque, _pad;
} gor_rect;

/* sample_candidates planner.hpp:56-107: returns the count, < 0 on error
 * (-1 bad bounds/config, -2 budget exhausted, -3 degenerate look-at). */
int gor_sample_candidates(const double* bmin, const double* bmax, const gor_rect* rects,
                          int n_rects, const gor_planner* pc, uint64_t step_seed, gor_camera* out);
/* vis_coverage planner.hpp:155-184 */
double gor_vis_coverage(const gor_rect* rects, int n_rects, double density, const gor_camera* views,
                        int n_views);

/* oracle.hpp:70-103 */
double gor_raymarch_transmittance(const gor_scene* s, const double* origin,
                                  const double* target, double step, int64_t exclude,
                                  double alpha_clamp_max);

#ifdef __cplusplus
}
#endif
#endif
