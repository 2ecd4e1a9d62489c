/*
 * gavis_b200.h -- C ABI of the B200-native GAVIS hot paths.
 *
 * Drop-in boundary for the two data-parallel paths of the GAVIS reference
 * (R/ = /root/reference/proj/include/gavis/):
 *   VF CONST   construct_field      vfield.hpp:68-92
 *              accumulate_view      vfield.hpp:38-63
 *              single_view_visibility raster.hpp:237-290
 *   VF QUERY   query_visibility     vfield.hpp:96-112
 *              query_view           vfield.hpp:121-134
 *   UA RENDER  render_entropy       uncertainty.hpp:242-260 (+ render_entropy_core :124-238)
 *              rasterize            raster.hpp:175-231
 *              image_entropy        uncertainty.hpp:264-278
 *              select_nbv           planner.hpp:117-137
 *
 * The reference has no FFI of its own: its boundary is the header-only C++ API
 * called by tools/gavis_main.cpp:79-80, :104-105 and planner.hpp:297-301.
 * include/gavis/gavis_b200.hpp re-exposes those exact C++ signatures on top of
 * this C ABI.
 *
 * Conventions
 *   - plain pointers and sizes; no CUDA or torch types in any signature;
 *   - every entry point returns a gavis_status; on failure gavis_last_error()
 *     holds a thread-local message. Status codes mirror the reference's
 *     exception taxonomy (common.hpp:22-46, exit codes gavis_main.cpp:358-371);
 *   - host output buffers are caller-owned; a NULL output pointer skips that
 *     output; calls are synchronous at the ABI;
 *   - scene arrays are fp32 (BASELINE.json configs); every decision on the path
 *     (projection, culling, tile keys, coverage, alpha, transmittance and the
 *     early-termination test) is computed in fp64 like the reference;
 *   - outputs are double, the reference's own type.
 */
#ifndef GAVIS_B200_H
#define GAVIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GAVIS_ABI_VERSION 1

typedef enum {
  GAVIS_OK = 0,
  GAVIS_ERR_PARAMETER = 2, /* ParameterError  (common.hpp:25-28) */
  GAVIS_ERR_INVARIANT = 3, /* InvariantError  (common.hpp:30-33) */
  GAVIS_ERR_ORACLE = 4,    /* OracleError     (common.hpp:35-38) */
  GAVIS_ERR_DEVICE = 5     /* CUDA / NCCL failure                 */
} gavis_status;

/* CameraView (model.hpp:66-105). rotation is row-major camera-to-world with
 * columns = camera x (image right), y (image down), z (forward). */
typedef struct {
  double rotation[9];
  double position[3];
  int32_t width, height;
  double fov_h, fov_v, near_plane;
} gavis_camera;

/* RasterConfig (raster.hpp:21-35). Defaults 16 / 1e-4 / 0.3 / 0.99. */
typedef struct {
  int32_t tile_size;
  int32_t _pad;
  double transmittance_cutoff, dilation, alpha_clamp_max;
} gavis_raster_config;

/* UncertaintyConfig (uncertainty.hpp:24-52). variance_provider: 0 kConstant,
 * 1 kShPropagation (needs gavis_scene_set_coeff_variances); correlation: 0 kNone,
 * 1 kHook (image score sum of H - H exp(-d / correlation_lambda), d the entropy
 * depth; lambda must be positive). */
typedef struct {
  double beta, prior_opacity, color_sigma;
  double prior_cov[9];
  int32_t variance_provider, correlation;
  double correlation_lambda;
} gavis_uncertainty_config;

/* Scene (model.hpp:130-134) as fp32 structure of arrays. */
typedef struct {
  int64_t num_particles;
  int32_t color_degree, _pad;
  const float* positions;    /* [N*3]                                     */
  const float* rotations;    /* [N*4] quaternion (w, x, y, z)             */
  const float* scales;       /* [N*3] per-axis standard deviations        */
  const float* opacities;    /* [N]                                       */
  const float* colors;       /* [N*3*(Lc+1)^2] per particle, channel-major */
  const uint8_t* is_virtual; /* [N] or NULL                               */
} gavis_scene_desc;

typedef struct gavis_ctx gavis_ctx;
typedef struct gavis_scene gavis_scene;
typedef struct gavis_field gavis_field;

/* ---- runtime ---------------------------------------------------------- */
int gavis_abi_version(void);
const char* gavis_last_error(void);
/* One context per device (one process per GPU). stream: a cudaStream_t passed
 * as void* to run on the caller's stream, or NULL for a private stream. */
gavis_status gavis_ctx_create(int32_t device, void* stream, gavis_ctx** out);
gavis_status gavis_ctx_destroy(gavis_ctx* ctx);
gavis_status gavis_ctx_synchronize(gavis_ctx* ctx);
/* Views processed per launch batch (0 = automatic from free memory). */
gavis_status gavis_ctx_set_batch(gavis_ctx* ctx, int32_t max_views_per_batch);
/* Tile pairs one batch may hold (0 = automatic: the batch memory budget / 32 B,
 * at most 2^31 - 1). A batch of views whose pairs exceed it is re-binned with
 * half the views (down to one view; one view may produce up to 2^31 - 1 pairs). */
gavis_status gavis_ctx_set_pair_budget(gavis_ctx* ctx, int64_t max_pairs_per_batch);
/* Arithmetic of the UA render (gavis_ua_render, gavis_select_nbv, loops):
 *  GAVIS_PRECISION_EXACT (default): every blend in fp64 (alpha, both
 *    transmittances, stop tests, accumulations; FMA-contracted, to rounding of
 *    the reference's unfused double code); the SH colour dot product on the
 *    tensor cores in split fp16 (~2^-21 relative). Images to ~1e-7 of the
 *    reference, entropy and scores to ~1e-13.
 *  GAVIS_PRECISION_CERTIFIED: fp32 blend with a per-pixel error bound on the
 *    early-termination tests; pixels the bound cannot certify are recomputed
 *    in fp64, so contributor counts equal the fp64 reference's; images agree
 *    with it to ~1e-6 (north_star: 1e-4); select_nbv re-scores in fp64 every
 *    candidate whose score interval (rigorous per-candidate error bounds,
 *    gavis_ctx_last_score_bounds) can reach the best's, so the argmax is the
 *    fp64 one. Used for 16x16 tiles and alpha_clamp_max <= 0.999, scenes with
 *    opacities >= 0 and visibilities in [0, 1] (other inputs, and scoring calls
 *    with the correlation hook or sh_propagation, which have no score bound,
 *    run the fp64 path). */
enum { GAVIS_PRECISION_CERTIFIED = 0, GAVIS_PRECISION_EXACT = 1 };
gavis_status gavis_ctx_set_precision(gavis_ctx* ctx, int32_t precision);
/* Rigorous per-candidate bounds on |certified score - fp64 score| of the last
 * scored render or select_nbv on this context (certified mode, constant variance
 * provider, no correlation hook; see kernels_ua_fast.cu "score bound"): *n_out =
 * 0 when it had none. select_nbv re-scores in fp64 every candidate i with
 * s_i >= s_best - max(e_best + e_i, 1e-3 |s_best|, 1e-9). */
gavis_status gavis_ctx_last_score_bounds(gavis_ctx* ctx, double* bounds, int32_t capacity,
                                         int32_t* n_out);
/* Counters since context creation: pixels recomputed in fp64 by the certified
 * blend, candidates re-scored in fp64 to certify an argmax. Either may be NULL. */
gavis_status gavis_ctx_get_counters(gavis_ctx* ctx, int64_t* redo_pixels,
                                    int64_t* rescored_views);
/* Per-kernel CUDA-event timing on the context stream (off by default). */
gavis_status gavis_ctx_set_profiling(gavis_ctx* ctx, int32_t enabled);
/* Accumulated device milliseconds and launch count of a kernel family:
 * "preprocess", "emit_keys", "sort", "ranges", "vf_blend", "vf_finalize",
 * "ua_blend", "ua_redo", "score", "query". Resets when reset != 0. */
gavis_status gavis_ctx_kernel_time(gavis_ctx* ctx, const char* kernel, double* ms,
                                   int64_t* launches, int32_t reset);
/* Device-side stopwatch on the context stream (bench timing). */
gavis_status gavis_ctx_timer_start(gavis_ctx* ctx);
gavis_status gavis_ctx_timer_stop(gavis_ctx* ctx, double* ms);
/* Total kernels launched by this context since creation. */
gavis_status gavis_ctx_launch_count(gavis_ctx* ctx, int64_t* launches);

/* ---- scene ------------------------------------------------------------ */
gavis_status gavis_scene_upload(gavis_ctx* ctx, const gavis_scene_desc* desc,
                                gavis_scene** out);
gavis_status gavis_scene_destroy(gavis_scene* scene);
/* Per-particle per-channel SH coefficient variances [N][3][(Lv+1)^2] for the
 * sh_propagation variance provider (UncertaintyConfig::coeff_variances,
 * uncertainty.hpp:38, :63-83). Lv <= 4; negative entries -> PARAMETER. */
gavis_status gavis_scene_set_coeff_variances(gavis_ctx* ctx, gavis_scene* scene,
                                             const float* variances, int32_t degree);
gavis_status gavis_scene_num_particles(const gavis_scene* scene, int64_t* n);

/* ---- visibility field (vfield.hpp) ------------------------------------ */
/* construct_field (vfield.hpp:68-92): zeroed field, every view rendered, SH
 * accumulated in trajectory order, num_views = n_views. */
gavis_status gavis_vf_construct(gavis_ctx* ctx, const gavis_scene* scene,
                                const gavis_camera* views, int32_t n_views, double kappa,
                                int32_t degree, const gavis_raster_config* rc,
                                gavis_field** out);
/* An all-zero field (num_views = 0) to accumulate into. */
gavis_status gavis_vf_create(gavis_ctx* ctx, const gavis_scene* scene, double kappa,
                             int32_t degree, gavis_field** out);
/* Renders and accumulates views into an existing field in order; adds n_views
 * to num_views (incremental / sharded construction, vfield.hpp:38-63, :88-90). */
gavis_status gavis_vf_accumulate_views(gavis_ctx* ctx, gavis_field* field,
                                       const gavis_scene* scene, const gavis_camera* views,
                                       int32_t n_views, const gavis_raster_config* rc);
/* accumulate_view with caller-provided per-particle visibility [N]. */
gavis_status gavis_vf_accumulate_visibility(gavis_ctx* ctx, gavis_field* field,
                                            const gavis_scene* scene,
                                            const gavis_camera* view, const double* visibility);
/* Field from host coefficients (e.g. a field.json written by the reference). */
gavis_status gavis_vf_upload(gavis_ctx* ctx, const gavis_scene* scene, double kappa,
                             int32_t degree, int32_t num_views, const double* gamma,
                             gavis_field** out);
gavis_status gavis_vf_download(const gavis_field* field, double* gamma, int32_t* num_views,
                               int32_t* degree);
gavis_status gavis_vf_set_num_views(gavis_field* field, int32_t num_views);
/* Device pointer and element count of gamma (float64, N*(L+1)^2 row-major) for
 * an in-place NCCL all-reduce of per-rank partial fields. */
gavis_status gavis_vf_device_gamma(gavis_field* field, void** device_ptr, int64_t* count);
gavis_status gavis_vf_destroy(gavis_field* field);

/* single_view_visibility (raster.hpp:237-290): v [N]; optional touch counts [N]
 * and per-pixel contributor counts [W*H]. */
gavis_status gavis_single_view_visibility(gavis_ctx* ctx, const gavis_scene* scene,
                                          const gavis_camera* cam,
                                          const gavis_raster_config* rc, double* visibility,
                                          int64_t* touch, int32_t* contributors);

/* query_visibility (vfield.hpp:96-112) for n (particle, direction) pairs. */
gavis_status gavis_vf_query(gavis_ctx* ctx, const gavis_field* field,
                            const int64_t* particle_index, const double* directions,
                            int64_t n, double* visibility);
/* query_view (vfield.hpp:121-134): non-culled particles in index order. */
gavis_status gavis_vf_query_view(gavis_ctx* ctx, const gavis_field* field,
                                 const gavis_scene* scene, const gavis_camera* cam,
                                 double dilation, int32_t* particle_index, double* visibility,
                                 int64_t* n_out);

/* ---- uncertainty-aware render (uncertainty.hpp, raster.hpp) ------------- */
/* Fused render of n cameras (all outputs nullable, laid out camera-major):
 *   rgb [n*H*W*3], depth [n*H*W], transmittance [n*H*W]   -- rasterize
 *   entropy [n*H*W], invisible_mass [n*H*W], entropy_depth [n*H*W]
 *                                                         -- render_entropy
 *   scores [n]                                            -- image_entropy
 * field == NULL with splat_visibility != NULL runs render_entropy_core with
 * caller-provided per-particle visibility [N] (one vector for all cameras).
 * If every image pointer is NULL but scores is set, images are not written
 * back (device-resident), but RGB is still composited when with_rgb != 0. */
typedef struct {
  double* rgb;
  double* depth;
  double* transmittance;
  double* entropy;
  double* invisible_mass;
  double* entropy_depth;
  double* scores;
  int32_t* rgb_contributors;     /* per-pixel covered entries, RGB track  */
  int32_t* entropy_contributors; /* per-pixel covered entries, entropy track */
  int32_t with_rgb;              /* composite RGB even if rgb == NULL       */
  int32_t with_entropy;          /* composite entropy even if entropy == NULL */
} gavis_render_outputs;

gavis_status gavis_ua_render(gavis_ctx* ctx, const gavis_scene* scene,
                             const gavis_field* field, const double* splat_visibility,
                             const gavis_camera* cams, int32_t n_cams,
                             const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                             gavis_render_outputs* out);

/* render_entropy's mixtures_out (uncertainty.hpp:90-102, :207-230) for one
 * camera: the components of every pixel (composited entries with w* > 0, in
 * compositing order) in CSR form. offsets [W*H+1] is always written;
 * components are written when non-NULL and capacity >= offsets[W*H] (call once
 * with components = NULL to size the buffer). prior_weight (w0),
 * residual_transmittance (T*) and entropy per pixel are optional. Field or
 * splat_visibility as in gavis_ua_render. Computed with the exact fp64 track. */
typedef struct {
  double weight;  /* w* = alpha* T */
  double vis;     /* particle visibility v */
  double mean[3]; /* clamped SH colour at the pixel ray */
  double var[3];  /* diagonal of Q_c */
} gavis_mixture_component;

gavis_status gavis_ua_mixtures(gavis_ctx* ctx, const gavis_scene* scene, const gavis_field* field,
                               const double* splat_visibility, const gavis_camera* cam,
                               const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                               int64_t* offsets, gavis_mixture_component* components,
                               int64_t capacity, double* prior_weight,
                               double* residual_transmittance, double* entropy);

/* select_nbv (planner.hpp:117-137): scores [n] and the first maximum. */
gavis_status gavis_select_nbv(gavis_ctx* ctx, const gavis_scene* scene,
                              const gavis_field* field, const gavis_camera* cams,
                              int32_t n_cams, const gavis_raster_config* rc,
                              const gavis_uncertainty_config* uc, int32_t with_rgb,
                              double* scores, int32_t* best_index);

/* Greedy NBV loop with incremental field updates (run_active_mapping,
 * planner.hpp:284-316, with density control off): for each of `steps` rounds,
 * select_nbv over the candidate pool, append the chosen camera to the field by
 * accumulating its view (gamma is linear in the views, vfield.hpp:53-60), and
 * record chosen index and score. chosen[steps], scores[steps] (nullable),
 * all_scores[steps * n_cams] (nullable). */
gavis_status gavis_nbv_loop(gavis_ctx* ctx, const gavis_scene* scene, gavis_field* field,
                            const gavis_camera* cams, int32_t n_cams, int32_t steps,
                            const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                            int32_t with_rgb, int32_t* chosen, double* scores,
                            double* all_scores);

/* ---- multi-GPU: one process per GPU over NCCL -------------- */
/* The reference parallelises construct_field over views (vfield.hpp:85-90) and
 * select_nbv over candidates (planner.hpp:125-131) with static blocks
 * (parallel.hpp:35-60); these entry points apply the same blocks across ranks.
 * NCCL is loaded at run time (libnccl.so.2; the process's own copy if one is
 * already loaded). Communicator: rank 0 calls gavis_comm_unique_id, the caller
 * ships the GAVIS_COMM_ID_BYTES bytes to every rank (MPI, a file, a socket),
 * and every rank calls gavis_comm_create with its own context; or an existing
 * ncclComm_t is wrapped with gavis_comm_adopt (not destroyed with the comm). */
#define GAVIS_COMM_ID_BYTES 128
typedef struct gavis_comm gavis_comm;
gavis_status gavis_comm_unique_id(uint8_t* id_out /* [GAVIS_COMM_ID_BYTES] */);
gavis_status gavis_comm_create(gavis_ctx* ctx, const uint8_t* id, int32_t nranks, int32_t rank,
                               gavis_comm** out);
gavis_status gavis_comm_adopt(gavis_ctx* ctx, void* nccl_comm, int32_t nranks, int32_t rank,
                              gavis_comm** out);
gavis_status gavis_comm_destroy(gavis_comm* comm);
/* In-place sum of a field's fp64 coefficients over the ranks (ncclAllReduce on
 * the context stream): partial fields of disjoint view blocks -> the full field. */
gavis_status gavis_vf_allreduce(gavis_comm* comm, gavis_field* field);
/* construct_field (vfield.hpp:68-92) with the views split in static blocks over
 * the ranks: each rank renders [n*r/w, n*(r+1)/w), the partials are all-reduced,
 * num_views = n_views on every rank. Collective: every rank calls it. */
gavis_status gavis_vf_construct_sharded(gavis_comm* comm, const gavis_scene* scene,
                                        const gavis_camera* views, int32_t n_views, double kappa,
                                        int32_t degree, const gavis_raster_config* rc,
                                        gavis_field** out);
/* select_nbv (planner.hpp:117-137) over the full candidate list, each rank
 * scoring its static block; scores [n_cams] (all of them, on every rank) and
 * the first maximum. Certified mode re-scores the contenders of the maximum in
 * fp64 on their owning ranks. Collective: every rank calls it. */
gavis_status gavis_select_nbv_sharded(gavis_comm* comm, const gavis_scene* scene,
                                      const gavis_field* field, const gavis_camera* cams,
                                      int32_t n_cams, const gavis_raster_config* rc,
                                      const gavis_uncertainty_config* uc, int32_t with_rgb,
                                      double* scores, int32_t* best_index);

/* ---- density control (vfield.hpp:136-199) ------------------------------ */
/* DensityControlConfig (vfield.hpp:136-147). Defaults rho 100, eta 0.5,
 * eps_v 0.95, seed 0. */
typedef struct {
  double rho, eta, eps_v;
  uint64_t seed;
} gavis_density_config;

/* density_control: floor(rho * volume(bounds)) transparent virtual probes
 * (SplitMix64(derive_seed(seed, k)) positions, scale cbrt(3(1+eta)/(4 pi rho)),
 * stored in fp32 like every scene array), isotropic multi-view visibility
 * 1 - prod_views(1 - b) computed on the device with the VF kernels, probes with
 * visibility <= eps_v appended after the real particles in a new device scene
 * (*out, caller destroys). kept_ids (nullable, capacity kept_capacity) receives
 * the probe indices k in sampling order. */
gavis_status gavis_density_control(gavis_ctx* ctx, const gavis_scene* scene,
                                   const double* bounds_min, const double* bounds_max,
                                   const gavis_camera* views, int32_t n_views,
                                   const gavis_density_config* cfg,
                                   const gavis_raster_config* rc, gavis_scene** out,
                                   int64_t* n_kept, int64_t* kept_ids, int64_t kept_capacity);

/* ---- planner (planner.hpp; host C++ around the device entry points) ------ */
/* OccluderRect (model.hpp:141-150): corner + u edge_u + v edge_v, u, v in [0,1]. */
typedef struct {
  double corner[3], edge_u[3], edge_v[3];
  int32_t opaque;
  int32_t _pad;
} gavis_occluder_rect;

/* PlannerConfig (planner.hpp:24-42). mode: 0 kSe3, 1 kSe2. Defaults 0, 128,
 * 1.5, 10, 0, look_inward 1, clearance 0.1, 128x128, fov pi/2 x pi/2, near 0.05. */
typedef struct {
  int32_t mode, num_candidates;
  double se2_height;
  int32_t steps, look_inward;
  uint64_t seed;
  double clearance;
  int32_t cam_width, cam_height;
  double fov_h, fov_v, cam_near;
} gavis_planner_config;

/* MappingContext (planner.hpp:255-262): vmf kappa (default 1), field degree
 * (default 2), raster / uncertainty / density configs, density_enabled
 * (default 1). */
typedef struct {
  double kappa;
  int32_t field_degree, density_enabled;
  gavis_raster_config raster;
  gavis_uncertainty_config uncertainty;
  gavis_density_config density;
} gavis_mapping_config;

/* sample_candidates (planner.hpp:56-107), host only: rejection-sampled poses
 * from SplitMix64(derive_seed(step_seed, 0xca4d1d)), discarded within
 * `clearance` of an opaque rectangle; out[num_candidates]. Budget exhaustion
 * (100 draws per candidate) -> PARAMETER. */
gavis_status gavis_sample_candidates(const double* bounds_min, const double* bounds_max,
                                     const gavis_occluder_rect* rects, int32_t n_rects,
                                     const gavis_planner_config* pc, uint64_t step_seed,
                                     gavis_camera* out);

/* vis_coverage (planner.hpp:155-184), host only: area-weighted fraction of
 * occluder surface (sample_density samples per unit area) seen by a view. */
gavis_status gavis_vis_coverage(const gavis_occluder_rect* rects, int32_t n_rects,
                                double sample_density, const gavis_camera* views,
                                int32_t n_views, double* coverage);

/* run_active_mapping (planner.hpp:284-316): per step, density control
 * reseeded with derive_seed(density.seed, step) over the current trajectory
 * (if enabled), a field rebuilt on the augmented scene, candidates from
 * gavis_sample_candidates(bounds, ..., derive_seed(pc.seed, step)), select_nbv
 * (entropy only), the chosen view appended. Per step outputs (nullable):
 * chosen_views[steps], chosen_index[steps], chosen_score[steps],
 * all_scores[steps * num_candidates], vis_coverage[steps] (needs occluders),
 * mean_entropy[steps] = score / (width * height). */
gavis_status gavis_active_mapping(gavis_ctx* ctx, const gavis_scene* scene,
                                  const double* bounds_min, const double* bounds_max,
                                  const gavis_occluder_rect* rects, int32_t n_rects,
                                  double sample_density, const gavis_camera* init_views,
                                  int32_t n_init, const gavis_planner_config* pc,
                                  const gavis_mapping_config* mc, gavis_camera* chosen_views,
                                  int32_t* chosen_index, double* chosen_score,
                                  double* all_scores, double* vis_coverage,
                                  double* mean_entropy);

/* ---- on-disk formats (host only; io.hpp) -------------------------------- */
/* load_splat_ply (io.hpp:493-637), two-phase: gavis_ply_info gives the vertex
 * count and the colour degree implied by f_rest_*; gavis_read_splat_ply fills
 * caller arrays laid out like gavis_scene_desc (activations applied: sigmoid
 * opacity, exp scale, normalised quaternion, DC + 0.5/Y00) and the particle
 * AABB as bounds. Malformed files -> PARAMETER. */
gavis_status gavis_ply_info(const char* path, int64_t* n, int32_t* color_degree);
gavis_status gavis_read_splat_ply(const char* path, int64_t capacity, float* positions,
                                  float* rotations, float* scales, float* opacities,
                                  float* colors, double* bounds_min, double* bounds_max);
/* save_field / load_field (io.hpp:255-295): {"L", "kappa", "num_views",
 * "gamma" (one row of (L+1)^2 per particle), "virtual"}. Read is two-phase
 * (gamma == NULL first to get the row count). */
gavis_status gavis_field_json_write(const char* path, int32_t degree, double kappa,
                                    int32_t num_views, int64_t n, const double* gamma,
                                    const uint8_t* is_virtual);
gavis_status gavis_field_json_read(const char* path, int64_t capacity, int32_t* degree,
                                   double* kappa, int32_t* num_views, int64_t* n,
                                   double* gamma, uint8_t* is_virtual);

/* ---- parity / debug ----------------------------------------------------- */
/* Projection records of one camera (ImageSpaceSplat, raster.hpp:37-44) for all
 * N particles: culled[N] (1 = culled), mean[2N], conic[3N] (a, b, c), depth[N],
 * cover_rect[4N] (x0, x1, y0, y1: pixels whose centre passes splat_covers,
 * raster.hpp:97-99; empty when x0 > x1) and tile_rect[4N] (tx0, tx1, ty0, ty1
 * from covered_pixel_range, raster.hpp:138-159; empty when tx0 > tx1). */
gavis_status gavis_debug_project(gavis_ctx* ctx, const gavis_scene* scene,
                                 const gavis_camera* cam, double dilation, int32_t tile_size,
                                 uint8_t* culled, double* mean, double* conic, double* depth,
                                 int32_t* cover_rect, int32_t* tile_rect);
/* Sorted (tile, depth) keys of one camera: keys[K], particle ids[K] and the
 * tile ranges[2*tiles]. Call with keys == NULL to get K in *n_pairs. */
gavis_status gavis_debug_binning(gavis_ctx* ctx, const gavis_scene* scene,
                                 const gavis_camera* cam, const gavis_raster_config* rc,
                                 uint64_t* keys, int32_t* particle_ids, int64_t* ranges,
                                 int64_t* n_pairs);

#ifdef __cplusplus
}
#endif
#endif /* GAVIS_B200_H */
