// ua_host.cu -- uncertainty-aware render (render_entropy / rasterize,
// uncertainty.hpp:242-260, raster.hpp:175-231), image scores (:264-278) and
// select_nbv (planner.hpp:117-137) behind the C ABI: the three-stream batch
// pipeline, the certified blend + fp64 redo, the exact re-scoring of contenders.
#include "host.h"

namespace gavis {
namespace host {

// Certification window of the fp32 blend, relative to the cutoff: twice the
// bound u (16 + 3.2 k + 22 S) derived in kernels_ua_fast.cu (k composited
// entries, S = sum a/(1-a) over them).
// Opacities above 1 (not excluded by the reference) weaken the alpha-error
// bounds (q <= 2 ln(o_max / a); A a (1.5 q + 8) <= 8 o_max A): the S coefficient
// becomes 22 o_max + 6 ln(o_max) (22 for o_max <= 1).
constexpr double kGaussEntropyHost = 4.256815599614018;  // uncertainty.hpp:19

void cert_window(UaBlendArgs* ua, float max_opacity) {
  const double u = std::ldexp(1.0, -24);
  const double om = std::max(1.0, (double)max_opacity);
  ua->cert_base = (float)(2.0 * u * 16.0);
  ua->cert_per_step = (float)(2.0 * u * 3.2);
  ua->cert_sum = (float)(2.0 * u * (22.0 * om + 6.0 * std::log(om)));
  ua->cert_per_step2 = (float)(2.0 * u * (1.004 + 3e-4 * std::log(om)));
  ua->cert_sum2 = (float)(2.0 * u * (41.0 + 3.0 * std::log(om)) * om);
  // test hook (tests/test_certified.py): hand every pixel to the fp64 redo
  const char* force = std::getenv("GAVIS_CERT_FORCE_REDO");
  if (force && force[0] == '1') ua->cert_base = 3.0e38f;
  // timing hook only (uncertified results): flag no pixel, to measure what the
  // redo costs the step
  if (force && force[0] == 'n') {
    ua->cert_base = ua->cert_per_step = ua->cert_sum = 0.0f;
    ua->cert_per_step2 = ua->cert_sum2 = 0.0f;
  }
}

void ua_render(gavis_ctx* c, const gavis_scene* s, const gavis_field* f, const double* vis_host,
               const gavis_camera* cams, int n, const gavis_raster_config* rc,
               const gavis_uncertainty_config* uc, gavis_render_outputs* out) {
  NvtxRange nvtx("UA render (render_entropy + rasterize, uncertainty.hpp:242-260)");
  validate_raster(rc);
  double hl_q0 = 0.0;
  validate_unc(uc, &hl_q0);
  require(cams != nullptr || n == 0, "cameras must not be null");
  require(out != nullptr, "render outputs must not be null");
  check_scene_field(c, s, f);
  for (int i = 0; i < n; ++i) validate_camera(cams[i]);
  const int64_t N = s->dev.n;
  const bool do_rgb = out->rgb || out->depth || out->transmittance || out->rgb_contributors ||
                      out->with_rgb;
  const bool do_ent = out->entropy || out->invisible_mass || out->entropy_depth || out->scores ||
                      out->entropy_contributors || out->with_entropy;
  if (!do_rgb && !do_ent) return;
  const double* vis_dev = nullptr;
  bool vis_outside_unit = false;  // selects the exact kernels' lower alpha* clamp
  if (!f) {
    require(vis_host != nullptr || N == 0 || !do_ent,
            "render needs a field or per-particle splat visibility");
    if (vis_host && N > 0) {
      double* d = (double*)c->buf("vis_given", sizeof(double) * N);
      CK(cudaMemcpyAsync(d, vis_host, sizeof(double) * N, cudaMemcpyHostToDevice, c->stream));
      vis_dev = d;
      for (int64_t i = 0; i < N && !vis_outside_unit; ++i)
        vis_outside_unit = !(vis_host[i] >= 0.0 && vis_host[i] <= 1.0);
    }
  }
  // negative (or NaN) opacities make alpha, hence A alpha + B, negative: the exact
  // kernels then need the lower alpha* clamp (LO), as for visibilities outside
  // [0, 1]; the certified blend assumes neither happens (its bounds and its
  // clamp-free alpha* rely on alpha, v in [0, 1]) and is not used for such inputs
  const bool outside = vis_outside_unit || !s->opacity_nonneg;
  vis_outside_unit = outside;
  const int bv = batch_views(c, N, n);
  const bool fast = c->precision == GAVIS_PRECISION_CERTIFIED && !outside &&
                    ua_fast_supported(rc->tile_size, rc->alpha_clamp_max);
  unsigned long long* redo_total = nullptr;
  if (fast) {
    redo_total = (unsigned long long*)c->buf("redo_total", sizeof(unsigned long long));
    CK(cudaMemsetAsync(redo_total, 0, sizeof(unsigned long long), c->stream));
  }
  if (out->scores && n > c->pin_scores_cap) {
    c->sync_all();
    if (c->pin_scores) CK(cudaFreeHost(c->pin_scores));
    if (c->pin_bounds) CK(cudaFreeHost(c->pin_bounds));
    c->pin_scores = c->pin_bounds = nullptr;
    c->pin_scores_cap = 0;
    CK(cudaMallocHost(&c->pin_scores, sizeof(double) * n));
    CK(cudaMallocHost(&c->pin_bounds, sizeof(double) * n));
    c->pin_scores_cap = n;
  }
  // certified scores carry a rigorous error bound (kernels_ua_fast.cu, "score
  // bound") for the constant variance provider without the correlation hook
  const bool bounded = fast && out->scores && uc->variance_provider == 0 && uc->correlation == 0;
  c->score_bounds.clear();
  cudaStream_t const side = fast ? c->side_hi : c->side;
  CK(cudaEventRecord(c->ev_done[0], c->stream));  // side / front work start after this point
  CK(cudaStreamWaitEvent(side, c->ev_done[0], 0));
  CK(cudaStreamWaitEvent(c->front, c->ev_done[0], 0));
  cudaStream_t main_stream = c->stream;
  struct BufsetReset {
    gavis_ctx* c;
    cudaStream_t main;
    ~BufsetReset() {
      c->bufset = 0;
      c->stream = main;
    }
  } reset{c, main_stream};
  int64_t pix_done = 0;
  int batch = 0;
  // buffer sets in rotation: batch k's binning reuses the set of batch k - nsets,
  // whose side-stream redo reads its binning outputs (A/B: GAVIS_BUFSETS=2)
  static const int nsets = [] {
    const char* e = std::getenv("GAVIS_BUFSETS");
    return (e && e[0] == '2') ? 2 : gavis_ctx::kSets;
  }();
  int bvv = bv;  // views per batch; halved for good when a batch holds too many pairs
  for (int v0 = 0, V = 0; v0 < n; v0 += V, ++batch) {
    V = std::min(bvv, n - v0);
    const int par = batch % nsets;
    c->bufset = par;
    // binning runs on the front stream, under the previous batch's blend; the
    // buffers of this set were last read by batch - nsets's side-stream work
    c->stream = c->front;
    if (batch >= nsets) CK(cudaStreamWaitEvent(c->front, c->ev_done[par], 0));
    BinOpts o;
    o.ua = do_ent;
    o.field = f;
    o.vis_given_dev = vis_dev;
    o.beta = uc->beta;
    o.o0b = uc->prior_opacity * (1.0 - uc->beta);
    o.hl_const = 3.0 * std::log(uc->color_sigma);  // 0.5 log(sigma^6), uncertainty.hpp:145
    int* err = nullptr;
    if (do_ent && uc->variance_provider == 1) {
      require(s->var != nullptr || s->dev.n == 0,
              "variance_provider sh_propagation requires coeff_variances");
      o.var = s->var;
      o.var_degree = s->var_degree;
      err = (int*)c->buf("err_flag", sizeof(int));
      CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
      o.err_flag = err;
    }
    Binned b = bin_batch(c, s, cams + v0, V, rc, o);
    while (b.overflow) {
      V = bvv = std::max(1, V / 2);
      b = bin_batch(c, s, cams + v0, V, rc, o);
    }
    if (err) {
      CK(cudaMemcpyAsync(c->pinned + 2, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      require(c->pinned[2] == 0, "propagated color variance must be positive");
    }
    CK(cudaEventRecord(c->ev_bin[par], c->front));
    c->stream = main_stream;
    CK(cudaStreamWaitEvent(c->stream, c->ev_bin[par], 0));
    const int64_t P = b.total_pix;
    UaBlendArgs ua;
    ua.scene = s->dev;
    ua.cams = b.dcams;
    ua.V = V;
    ua.total_tiles = b.total_tiles;
    ua.tile_size = rc->tile_size;
    ua.cutoff = rc->transmittance_cutoff;
    ua.amax = rc->alpha_clamp_max;
    ua.hl_qc = 3.0 * std::log(uc->color_sigma);
    ua.hl_q0 = hl_q0;
    ua.corr_lambda = uc->correlation == 1 ? uc->correlation_lambda : 0.0;
    ua.geo = b.geo;
    ua.ua = b.ua;
    ua.ranges = b.ranges;
    ua.vals = b.vals;
    ua.do_rgb = do_rgb;
    ua.do_ent = do_ent;
    ua.vis_outside_unit = vis_outside_unit;
    // The RGB and entropy images always land in device memory (host copies only
    // when requested; the score folds the entropy image); depth and
    // residual-transmittance maps only on request.
    if (do_rgb) {
      ua.rgb = (double*)c->buf("img_rgb", sizeof(double) * 3 * P);
      ua.depth = out->depth ? (double*)c->buf("img_depth", sizeof(double) * P) : nullptr;
      ua.trans = out->transmittance ? (double*)c->buf("img_trans", sizeof(double) * P) : nullptr;
      if (out->rgb_contributors) ua.rgb_contrib = (int32_t*)c->buf("img_nrgb", sizeof(int32_t) * P);
    }
    if (do_ent) {
      ua.entropy = (double*)c->buf("img_entropy", sizeof(double) * P);
      ua.w0 = (double*)c->buf("img_w0", sizeof(double) * P);
      ua.edepth = (out->entropy_depth || ua.corr_lambda > 0.0)
                      ? (double*)c->buf("img_edepth", sizeof(double) * P)
                      : nullptr;
      if (out->entropy_contributors)
        ua.ent_contrib = (int32_t*)c->buf("img_nent", sizeof(int32_t) * P);
    }
    if (fast && b.total_tiles > 0) {
      invariant(P < (int64_t(1) << 32), "too many pixels in one batch");
      ua.flag_list = (uint32_t*)c->buf("flag_list", sizeof(uint32_t) * P);
      ua.flag_count = (uint32_t*)c->buf("flag_count", sizeof(uint32_t));
      CK(cudaMemsetAsync(ua.flag_count, 0, sizeof(uint32_t), c->stream));
      cert_window(&ua, s->max_opacity);
      if (bounded) {
        ua.score_bound = (double*)c->buf("img_bound", sizeof(double) * P);
        const double u = std::ldexp(1.0, -24);
        const double cabs = std::fabs(ua.hl_qc + kGaussEntropyHost);
        ua.w0_tail = 1.7e-3 * u * std::max(1.0, (double)s->max_opacity);
        ua.bound_tail = ua.w0_tail * (cabs + 89.0);
        ua.c0_abs = std::fabs(hl_q0 + kGaussEntropyHost);
        ua.c_ent = ua.hl_qc + kGaussEntropyHost;
      }
      c->run("ua_blend", [&] { launch_ua_blend_fast(ua, c->stream); });
      CK(cudaEventRecord(c->ev_blend[par], c->stream));
      CK(cudaStreamWaitEvent(side, c->ev_blend[par], 0));
      c->run("ua_redo", [&] { launch_ua_redo(ua, side); }, 1, side);
      launch_add_count(redo_total, ua.flag_count, side);
    } else {
      c->run("ua_blend", [&] { launch_ua_blend(ua, c->stream); }, b.total_tiles > 0 ? 1 : 0);
      CK(cudaEventRecord(c->ev_blend[par], c->stream));
      CK(cudaStreamWaitEvent(side, c->ev_blend[par], 0));
    }
    double* dscores = nullptr;
    double* dbounds = nullptr;
    if (do_ent) {
      dscores = (double*)c->buf("scores", sizeof(double) * V);
      double* part = (double*)c->buf("score_partial", sizeof(double) * V * score_partials_per_view());
      c->run("score", [&] {
        launch_score_image(b.dcams, V, ua.entropy, ua.edepth, ua.corr_lambda, part, dscores, side);
      }, 1, side);
      if (ua.score_bound) {  // the bound image folds like the score (fixed order)
        dbounds = (double*)c->buf("score_bounds", sizeof(double) * V);
        double* bpart = (double*)c->buf("bound_partial", sizeof(double) * V * score_partials_per_view());
        c->run("score", [&] {
          launch_score_image(b.dcams, V, ua.score_bound, nullptr, 0.0, bpart, dbounds, side);
        }, 1, side);
      }
    }
    copy_out(c, out->rgb ? out->rgb + 3 * pix_done : nullptr, ua.rgb, 3 * P, side);
    copy_out(c, out->depth ? out->depth + pix_done : nullptr, ua.depth, P, side);
    copy_out(c, out->transmittance ? out->transmittance + pix_done : nullptr, ua.trans, P, side);
    copy_out(c, out->entropy ? out->entropy + pix_done : nullptr, ua.entropy, P, side);
    copy_out(c, out->invisible_mass ? out->invisible_mass + pix_done : nullptr, ua.w0, P, side);
    copy_out(c, out->entropy_depth ? out->entropy_depth + pix_done : nullptr, ua.edepth, P, side);
    // scores through pinned staging: a D2H copy into pageable memory would block
    // the host on this batch's side-stream work and serialise the batches
    copy_out(c, out->scores ? c->pin_scores + v0 : nullptr, dscores, V, side);
    copy_out(c, dbounds ? c->pin_bounds + v0 : nullptr, dbounds, V, side);
    if (out->rgb_contributors)
      CK(cudaMemcpyAsync(out->rgb_contributors + pix_done, ua.rgb_contrib, sizeof(int32_t) * P,
                         cudaMemcpyDeviceToHost, side));
    if (out->entropy_contributors)
      CK(cudaMemcpyAsync(out->entropy_contributors + pix_done, ua.ent_contrib,
                         sizeof(int32_t) * P, cudaMemcpyDeviceToHost, side));
    CK(cudaEventRecord(c->ev_done[par], side));
    pix_done += P;
  }
  c->bufset = 0;
  // the main stream continues after the side stream's last batch
  CK(cudaEventRecord(c->ev_done[0], side));
  CK(cudaStreamWaitEvent(c->stream, c->ev_done[0], 0));
  if (redo_total) {
    CK(cudaMemcpyAsync(c->pinned + kPinRedo, redo_total, sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, c->stream));
  }
  c->sync_all();
  if (out->scores && n > 0) std::memcpy(out->scores, c->pin_scores, sizeof(double) * n);
  if (bounded && n > 0) {
    // fp64 folds of non-negative terms: relative rounding far below 1e-12
    c->score_bounds.assign(c->pin_bounds, c->pin_bounds + n);
    for (double& bd : c->score_bounds) bd *= 1.0 + 1e-12;
  }
  if (redo_total) c->redo_pixels += (int64_t)*reinterpret_cast<unsigned long long*>(c->pinned + kPinRedo);
}

// select_nbv's argmax (planner.hpp:132-136: first strictly greater score) over
// scores from the certified fp32 blend: every candidate i with
// s_i >= s_best - max(e_best + e_i, kCertScoreRel |s_best|, kCertScoreAbs), e the
// rigorous per-candidate score bounds K8 folds from K7f's per-pixel bounds, is
// re-scored with the exact fp64 blend and the argmax is taken again, so it is the
// exact path's argmax. (Scoring calls in the modes without a bound -- the
// correlation hook, sh_propagation -- run the fp64 path: ScoringPrecision, host.h.)
constexpr double kCertScoreRel = 1e-3;
constexpr double kCertScoreAbs = 1e-9;  // absolute floor: scores near 0 keep a window

std::vector<int> certified_contenders(gavis_ctx* c, const gavis_scene* s, const gavis_raster_config* rc,
                                      const std::vector<double>& sc) {
  std::vector<int> cont;
  // the same decision as ua_render's `fast` for a field render (identical on every
  // rank: the sharded select's re-scoring is collective)
  if (sc.empty() || c->precision != GAVIS_PRECISION_CERTIFIED || !s->opacity_nonneg ||
      !ua_fast_supported(rc->tile_size, rc->alpha_clamp_max))
    return cont;
  int b = 0;
  for (int i = 1; i < (int)sc.size(); ++i)
    if (sc[i] > sc[b]) b = i;
  // candidate i can hold the fp64 maximum only if s_i + e_i >= s_b - e_b, with
  // e the rigorous per-view bounds of the certified scores (when available);
  // the window is never narrower than kCertScoreRel |s_b| nor kCertScoreAbs
  const bool have = c->score_bounds.size() == sc.size();
  for (int i = 0; i < (int)sc.size(); ++i) {
    const double bound = have ? c->score_bounds[b] + c->score_bounds[i] : 0.0;
    const double window = std::max({bound, kCertScoreRel * std::fabs(sc[b]), kCertScoreAbs});
    if (sc[i] >= sc[b] - window) cont.push_back(i);
  }
  return cont;
}

int certified_first_max(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                        const gavis_camera* cams, int n, const gavis_raster_config* rc,
                        const gavis_uncertainty_config* uc, std::vector<double>& sc) {
  auto first_max = [&] {
    int b = 0;
    for (int i = 1; i < n; ++i)
      if (sc[i] > sc[b]) b = i;
    return b;
  };
  const std::vector<int> cont = certified_contenders(c, s, rc, sc);
  if (cont.size() < 2) return first_max();
  std::vector<gavis_camera> cc;
  for (int i : cont) cc.push_back(cams[i]);
  std::vector<double> ex(cont.size());
  gavis_render_outputs o = {};
  o.scores = ex.data();
  const std::vector<double> bounds = c->score_bounds;  // the fp64 re-render must not clear them
  c->precision = GAVIS_PRECISION_EXACT;
  try {
    ua_render(c, s, f, nullptr, cc.data(), (int)cc.size(), rc, uc, &o);
  } catch (...) {
    c->precision = GAVIS_PRECISION_CERTIFIED;
    c->score_bounds = bounds;
    throw;
  }
  c->precision = GAVIS_PRECISION_CERTIFIED;
  c->score_bounds = bounds;
  for (size_t k = 0; k < cont.size(); ++k) sc[cont[k]] = ex[k];
  c->rescored_views += (int64_t)cont.size();
  return first_max();
}

}  // namespace host
}  // namespace gavis

extern "C" {

gavis_status gavis_ua_render(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                             const double* splat_visibility, const gavis_camera* cams,
                             int32_t n_cams, const gavis_raster_config* rc,
                             const gavis_uncertainty_config* uc, gavis_render_outputs* out) {
  return guard([&] {
    require(c && s, "null argument");
    require(n_cams >= 0, "camera count must be non-negative");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    ua_render(c, s, f, splat_visibility, cams, n_cams, rc, uc, out);
  });
}

gavis_status gavis_ua_mixtures(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                               const double* splat_visibility, const gavis_camera* cam,
                               const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                               int64_t* offsets, gavis_mixture_component* components,
                               int64_t capacity, double* prior_weight,
                               double* residual_transmittance, double* entropy) {
  return guard([&] {
    require(c && s && cam && rc && uc && offsets, "null argument");
    validate_raster(rc);
    double hl_q0 = 0.0;
    validate_unc(uc, &hl_q0);
    validate_camera(*cam);
    check_scene_field(c, s, f);
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    const int64_t N = s->dev.n;
    const int64_t P = (int64_t)cam->width * cam->height;
    BinOpts o;
    o.ua = true;
    o.field = f;
    if (!f) {
      require(splat_visibility != nullptr || N == 0,
              "mixtures need a field or per-particle splat visibility");
      if (N > 0) {
        double* d = (double*)c->buf("vis_given", sizeof(double) * N);
        CK(cudaMemcpyAsync(d, splat_visibility, sizeof(double) * N, cudaMemcpyHostToDevice,
                           c->stream));
        o.vis_given_dev = d;
      }
    }
    o.beta = uc->beta;
    o.o0b = uc->prior_opacity * (1.0 - uc->beta);
    o.hl_const = 3.0 * std::log(uc->color_sigma);
    int* err = nullptr;
    if (uc->variance_provider == 1) {
      require(s->var != nullptr || N == 0,
              "variance_provider sh_propagation requires coeff_variances");
      o.var = s->var;
      o.var_degree = s->var_degree;
      err = (int*)c->buf("err_flag", sizeof(int));
      CK(cudaMemsetAsync(err, 0, sizeof(int), c->stream));
      o.err_flag = err;
    }
    Binned b = bin_batch(c, s, cam, 1, rc, o);
    if (err) {
      CK(cudaMemcpyAsync(c->pinned + 2, err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      c->sync();
      require(c->pinned[2] == 0, "propagated color variance must be positive");
    }
    MixtureArgs m;
    m.scene = s->dev;
    m.cam = b.dcams;
    m.tile_size = rc->tile_size;
    m.cutoff = rc->transmittance_cutoff;
    m.amax = rc->alpha_clamp_max;
    m.hl_q0 = hl_q0;
    m.var_const = uc->color_sigma * uc->color_sigma;
    m.geo = b.geo;
    m.ua = b.ua;
    m.ranges = b.ranges;
    m.vals = b.vals;
    m.var = o.var;
    m.var_degree = o.var_degree;
    m.counts = (int64_t*)c->buf("mix_counts", sizeof(int64_t) * std::max<int64_t>(1, P));
    m.prior = (double*)c->buf("mix_prior", sizeof(double) * std::max<int64_t>(1, P));
    m.resid = (double*)c->buf("mix_resid", sizeof(double) * std::max<int64_t>(1, P));
    m.entropy = (double*)c->buf("mix_entropy", sizeof(double) * std::max<int64_t>(1, P));
    c->run("mixtures", [&] { launch_mixtures(m, P, c->stream); });
    std::vector<int64_t> cnt((size_t)P);
    if (P > 0)
      CK(cudaMemcpyAsync(cnt.data(), m.counts, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, c->stream));
    copy_out(c, prior_weight, m.prior, P);
    copy_out(c, residual_transmittance, m.resid, P);
    copy_out(c, entropy, m.entropy, P);
    c->sync();
    offsets[0] = 0;
    for (int64_t p = 0; p < P; ++p) offsets[p + 1] = offsets[p] + cnt[p];
    const int64_t K = offsets[P];
    if (components && K > 0) {
      require(capacity >= K, "mixtures: capacity is smaller than offsets[W*H]");
      int64_t* doff = (int64_t*)c->buf("mix_offsets", sizeof(int64_t) * (P + 1));
      CK(cudaMemcpyAsync(doff, offsets, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, c->stream));
      m.offsets = doff;
      m.comps = (double*)c->buf("mix_comps", sizeof(double) * 8 * K);
      c->run("mixtures", [&] { launch_mixtures(m, P, c->stream); });
      static_assert(sizeof(gavis_mixture_component) == 8 * sizeof(double), "component layout");
      CK(cudaMemcpyAsync(components, m.comps, sizeof(double) * 8 * K, cudaMemcpyDeviceToHost,
                         c->stream));
      c->sync();
    }
  });
}

gavis_status gavis_select_nbv(gavis_ctx* c, const gavis_scene* s, const gavis_field* f,
                              const gavis_camera* cams, int32_t n_cams,
                              const gavis_raster_config* rc, const gavis_uncertainty_config* uc,
                              int32_t with_rgb, double* scores, int32_t* best) {
  return guard([&] {
    require(c && s && f, "null argument");
    require(n_cams > 0 && cams != nullptr, "select_nbv: candidate list must be nonempty");
    std::lock_guard<std::recursive_mutex> lk(c->mu);
    c->use();
    NvtxRange nvtx("select_nbv (planner.hpp:117-137)");
    ScoringPrecision sp(c, uc);
    std::vector<double> sc((size_t)n_cams);
    gavis_render_outputs o = {};
    o.scores = sc.data();
    o.with_rgb = with_rgb;
    ua_render(c, s, f, nullptr, cams, n_cams, rc, uc, &o);
    const int b = certified_first_max(c, s, f, cams, n_cams, rc, uc, sc);
    if (scores) std::memcpy(scores, sc.data(), sizeof(double) * n_cams);
    if (best) *best = b;
  });
}

}  // extern "C"
