// ref_driver.cpp -- C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/gavis/*.hpp, compiled in place against the
// Eigen-subset shim oracle/eigen_shim). TEST INFRASTRUCTURE ONLY: the checker
// and the reference arm's CPU implementation, never the product.
//
// Built by oracle/Makefile into oracle/_ref/libgavis_ref.so when /root/reference
// exists; the .so travels to the GPU box with the snapshot (git-ignored only).
// Structs are the oracle's (gavis_oracle.h), so oracle.py's ctypes types serve.
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <gavis/planner.hpp>
#include <gavis/raster.hpp>
#include <gavis/uncertainty.hpp>
#include <gavis/vfield.hpp>

#include "gavis_oracle.h"

namespace {

thread_local std::string g_err;

gavis::Scene make_scene(const gor_scene* s) {
  gavis::Scene sc;
  sc.color_degree = s->color_degree;
  const int nb = (s->color_degree + 1) * (s->color_degree + 1);
  sc.particles.resize((size_t)s->num_particles);
  for (int64_t i = 0; i < s->num_particles; ++i) {
    gavis::GaussianParticle& p = sc.particles[(size_t)i];
    p.position = gavis::Vec3(s->positions[3 * i], s->positions[3 * i + 1], s->positions[3 * i + 2]);
    p.rotation = gavis::Quat(s->rotations[4 * i], s->rotations[4 * i + 1], s->rotations[4 * i + 2],
                             s->rotations[4 * i + 3]);  // (w, x, y, z), as stored: not renormalised
    p.scale = gavis::Vec3(s->scales[3 * i], s->scales[3 * i + 1], s->scales[3 * i + 2]);
    p.opacity = s->opacities[i];
    for (int c = 0; c < 3; ++c)
      p.color_sh[c].assign(s->colors + (i * 3 + c) * nb, s->colors + (i * 3 + c + 1) * nb);
    p.is_virtual = s->is_virtual ? s->is_virtual[i] != 0 : false;
  }
  return sc;
}

gavis::CameraView make_cam(const gor_camera* c) {
  gavis::CameraView v;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) v.rotation(r, k) = c->rotation[r * 3 + k];
  v.position = gavis::Vec3(c->position[0], c->position[1], c->position[2]);
  v.width = c->width;
  v.height = c->height;
  v.fov_h = c->fov_h;
  v.fov_v = c->fov_v;
  v.near = c->near_plane;
  return v;
}

gavis::RasterConfig make_rc(const gor_raster* r) {
  gavis::RasterConfig rc;
  rc.tile_size = r->tile_size;
  rc.transmittance_cutoff = r->transmittance_cutoff;
  rc.dilation = r->dilation;
  rc.alpha_clamp_max = r->alpha_clamp_max;
  return rc;
}

gavis::UncertaintyConfig make_uc(const gor_unc* u) {
  gavis::UncertaintyConfig uc;
  uc.beta = u->beta;
  uc.prior_opacity = u->prior_opacity;
  uc.color_sigma = u->color_sigma;
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) uc.prior_cov(r, k) = u->prior_cov[r * 3 + k];
  uc.correlation = u->correlation == 1 ? gavis::CorrelationMode::kHook : gavis::CorrelationMode::kNone;
  uc.correlation_lambda = u->correlation_lambda;
  return uc;
}

gavis::VisibilityField make_field(const gavis::Scene& sc, const double* gamma, int degree, int num_views) {
  gavis::VisibilityField f;
  f.degree = degree;
  f.num_views = num_views;
  f.num_particles = sc.particles.size();
  const size_t nb = (size_t)(degree + 1) * (degree + 1);
  f.gamma.assign(gamma, gamma + nb * f.num_particles);
  f.virtual_mask.resize(f.num_particles);
  for (size_t i = 0; i < f.num_particles; ++i) f.virtual_mask[i] = sc.particles[i].is_virtual ? 1 : 0;
  return f;
}

gavis::OccluderSet make_occluders(const gor_rect* rects, int n, double density) {
  gavis::OccluderSet occ;
  occ.sample_density = density;
  for (int i = 0; i < n; ++i) {
    gavis::OccluderRect r;
    r.corner = gavis::Vec3(rects[i].corner[0], rects[i].corner[1], rects[i].corner[2]);
    r.edge_u = gavis::Vec3(rects[i].edge_u[0], rects[i].edge_u[1], rects[i].edge_u[2]);
    r.edge_v = gavis::Vec3(rects[i].edge_v[0], rects[i].edge_v[1], rects[i].edge_v[2]);
    r.opaque = rects[i].opaque != 0;
    occ.rectangles.push_back(r);
  }
  return occ;
}

gavis::PlannerConfig make_pc(const gor_planner* p) {
  gavis::PlannerConfig pc;
  pc.mode = p->mode == 1 ? gavis::PoseMode::kSe2 : gavis::PoseMode::kSe3;
  pc.num_candidates = p->num_candidates;
  pc.se2_height = p->se2_height;
  pc.steps = p->steps;
  pc.seed = p->seed;
  pc.look_inward = p->look_inward != 0;
  pc.clearance = p->clearance;
  pc.cam_width = p->cam_width;
  pc.cam_height = p->cam_height;
  pc.fov_h = p->fov_h;
  pc.fov_v = p->fov_v;
  pc.cam_near = p->cam_near;
  return pc;
}

void put_cam(const gavis::CameraView& v, gor_camera* c) {
  for (int r = 0; r < 3; ++r)
    for (int k = 0; k < 3; ++k) c->rotation[r * 3 + k] = v.rotation(r, k);
  for (int k = 0; k < 3; ++k) c->position[k] = v.position[k];
  c->width = v.width;
  c->height = v.height;
  c->fov_h = v.fov_h;
  c->fov_v = v.fov_v;
  c->near_plane = v.near;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const gavis::ParameterError& e) {
    g_err = e.what();
    return 2;
  } catch (const gavis::InvariantError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

}  // namespace

extern "C" {

const char* gref_last_error(void) { return g_err.c_str(); }

// A reference Scene built once (the AoS of GaussianParticle with its per-channel
// colour vectors), so timed calls measure the reference's work, not the copy.
void* gref_scene_new(const gor_scene* s) {
  try {
    return new gavis::Scene(make_scene(s));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void gref_scene_free(void* h) { delete static_cast<gavis::Scene*>(h); }

// select_nbv + rasterize of every candidate (the bench step's work: scores and
// the RGB renders), on a prebuilt scene handle.
int gref_select_nbv_rgb_h(void* h, const double* gamma, int degree, int num_views, const gor_camera* cams,
                          int n, const gor_raster* rc, const gor_unc* u, int threads, double* scores,
                          int* best) {
  return guarded([&] {
    const gavis::Scene& sc = *static_cast<gavis::Scene*>(h);
    const gavis::VisibilityField f = make_field(sc, gamma, degree, num_views);
    std::vector<gavis::CameraView> cv;
    for (int i = 0; i < n; ++i) cv.push_back(make_cam(&cams[i]));
    const gavis::RasterConfig r = make_rc(rc);
    const gavis::NbvResult res = gavis::select_nbv(sc, f, cv, r, make_uc(u), threads);
    // RGB renders, parallel over candidates like select_nbv (planner.hpp:125-131)
    gavis::parallel_for(n, threads, [&](int i) { (void)gavis::rasterize(sc, cv[(size_t)i], r, 1); });
    std::memcpy(scores, res.scores.data(), sizeof(double) * res.scores.size());
    *best = res.best_index;
  });
}

// construct_field on a prebuilt scene handle
int gref_construct_field_h(void* h, const gor_camera* views, int n_views, double kappa, int degree,
                           const gor_raster* rc, int threads, double* gamma) {
  return guarded([&] {
    const gavis::Scene& sc = *static_cast<gavis::Scene*>(h);
    gavis::Trajectory traj;
    for (int i = 0; i < n_views; ++i) traj.views.push_back(make_cam(&views[i]));
    const gavis::VisibilityField f =
        gavis::construct_field(sc, traj, gavis::VmfParams(kappa), degree, make_rc(rc), threads);
    std::memcpy(gamma, f.gamma.data(), sizeof(double) * f.gamma.size());
  });
}

// single_view_visibility (raster.hpp:237-290) -> v[N]
int gref_single_view_visibility(const gor_scene* s, const gor_camera* cam, const gor_raster* rc, int threads,
                                double* v) {
  return guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const std::vector<double> out = gavis::single_view_visibility(sc, make_cam(cam), make_rc(rc), threads);
    std::memcpy(v, out.data(), sizeof(double) * out.size());
  });
}

// construct_field (vfield.hpp:68-92) -> gamma[N * (L+1)^2]
int gref_construct_field(const gor_scene* s, const gor_camera* views, int n_views, double kappa, int degree,
                         const gor_raster* rc, int threads, double* gamma) {
  return guarded([&] {
    const gavis::Scene sc = make_scene(s);
    gavis::Trajectory traj;
    for (int i = 0; i < n_views; ++i) traj.views.push_back(make_cam(&views[i]));
    const gavis::VisibilityField f =
        gavis::construct_field(sc, traj, gavis::VmfParams(kappa), degree, make_rc(rc), threads);
    std::memcpy(gamma, f.gamma.data(), sizeof(double) * f.gamma.size());
  });
}

// rasterize (raster.hpp:175-231) -> rgb[3P], depth[P], T[P]
int gref_rasterize(const gor_scene* s, const gor_camera* cam, const gor_raster* rc, int threads, double* rgb,
                   double* depth, double* trans) {
  return guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const gavis::RenderOutput r = gavis::rasterize(sc, make_cam(cam), make_rc(rc), threads);
    std::memcpy(rgb, r.color.data(), sizeof(double) * r.color.size());
    std::memcpy(depth, r.depth.data(), sizeof(double) * r.depth.size());
    std::memcpy(trans, r.transmittance.data(), sizeof(double) * r.transmittance.size());
  });
}

// render_entropy (uncertainty.hpp:242-260) -> H[P], w0[P], entropy depth[P]
int gref_render_entropy(const gor_scene* s, const double* gamma, int degree, int num_views, const gor_camera* cam,
                        const gor_raster* rc, const gor_unc* u, int threads, double* H, double* w0,
                        double* depth) {
  return guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const gavis::VisibilityField f = make_field(sc, gamma, degree, num_views);
    std::vector<double> d;
    const gavis::EntropyMap m =
        gavis::render_entropy(sc, f, make_cam(cam), make_rc(rc), make_uc(u), threads, &d);
    std::memcpy(H, m.entropy.data(), sizeof(double) * m.entropy.size());
    std::memcpy(w0, m.invisible_mass.data(), sizeof(double) * m.invisible_mass.size());
    if (depth) std::memcpy(depth, d.data(), sizeof(double) * d.size());
  });
}

// select_nbv (planner.hpp:117-137) -> scores[n], best index
int gref_select_nbv(const gor_scene* s, const double* gamma, int degree, int num_views, const gor_camera* cams,
                    int n, const gor_raster* rc, const gor_unc* u, int threads, double* scores, int* best) {
  return guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const gavis::VisibilityField f = make_field(sc, gamma, degree, num_views);
    std::vector<gavis::CameraView> cv;
    for (int i = 0; i < n; ++i) cv.push_back(make_cam(&cams[i]));
    const gavis::NbvResult r = gavis::select_nbv(sc, f, cv, make_rc(rc), make_uc(u), threads);
    std::memcpy(scores, r.scores.data(), sizeof(double) * r.scores.size());
    *best = r.best_index;
  });
}

// sample_candidates (planner.hpp:56-107) -> count written to out (-1 on error)
int gref_sample_candidates(const double* bmin, const double* bmax, const gor_rect* rects, int n_rects,
                           const gor_planner* pc, uint64_t step_seed, gor_camera* out) {
  int n = -1;
  const int st = guarded([&] {
    gavis::Bounds b;
    b.min = gavis::Vec3(bmin[0], bmin[1], bmin[2]);
    b.max = gavis::Vec3(bmax[0], bmax[1], bmax[2]);
    const auto cams = gavis::sample_candidates(b, make_occluders(rects, n_rects, 64.0), make_pc(pc), step_seed);
    for (size_t i = 0; i < cams.size(); ++i) put_cam(cams[i], &out[i]);
    n = (int)cams.size();
  });
  return st == 0 ? n : -st;
}

// vis_coverage (planner.hpp:155-184)
double gref_vis_coverage(const gor_rect* rects, int n_rects, double density, const gor_camera* views,
                         int n_views) {
  double cov = -1.0;
  guarded([&] {
    gavis::Trajectory t;
    for (int i = 0; i < n_views; ++i) t.views.push_back(make_cam(&views[i]));
    cov = gavis::vis_coverage(make_occluders(rects, n_rects, density), t);
  });
  return cov;
}

// density_control (vfield.hpp:157-199) -> the appended virtual particles'
// positions [m*3] (capacity cap), returns m (< 0 on error)
int64_t gref_density_control(const gor_scene* s, const double* bmin, const double* bmax,
                             const gor_camera* views, int n_views, double rho, double eta, double eps_v,
                             uint64_t seed, const gor_raster* rc, int threads, double* kept_pos, int64_t cap) {
  int64_t m = -1;
  const int st = guarded([&] {
    gavis::Scene sc = make_scene(s);
    sc.bounds.min = gavis::Vec3(bmin[0], bmin[1], bmin[2]);
    sc.bounds.max = gavis::Vec3(bmax[0], bmax[1], bmax[2]);
    gavis::Trajectory t;
    for (int i = 0; i < n_views; ++i) t.views.push_back(make_cam(&views[i]));
    gavis::DensityControlConfig cfg;
    cfg.rho = rho;
    cfg.eta = eta;
    cfg.eps_v = eps_v;
    cfg.seed = seed;
    const gavis::Scene out = gavis::density_control(sc, t, cfg, make_rc(rc), threads);
    m = (int64_t)(out.particles.size() - sc.particles.size());
    if (m > cap) throw gavis::InvariantError("density_control: kept_pos capacity too small");
    for (int64_t k = 0; k < m; ++k)
      for (int d = 0; d < 3; ++d) kept_pos[3 * k + d] = out.particles[sc.particles.size() + (size_t)k].position[d];
  });
  return st == 0 ? m : -st;
}

// run_active_mapping (planner.hpp:284-316) -> per step: chosen index, its score,
// vis_coverage, and all candidate scores [steps * num_candidates]
int gref_active_mapping(const gor_scene* s, const double* bmin, const double* bmax, const gor_rect* rects,
                        int n_rects, double density, const gor_camera* init, int n_init, const gor_planner* pc,
                        double kappa, int degree, const gor_raster* rc, const gor_unc* u, int density_enabled,
                        double rho, double eta, double eps_v, uint64_t dseed, int threads, int* chosen,
                        double* score, double* coverage, double* all_scores) {
  return guarded([&] {
    gavis::Scene sc = make_scene(s);
    sc.bounds.min = gavis::Vec3(bmin[0], bmin[1], bmin[2]);
    sc.bounds.max = gavis::Vec3(bmax[0], bmax[1], bmax[2]);
    gavis::Trajectory t;
    for (int i = 0; i < n_init; ++i) t.views.push_back(make_cam(&init[i]));
    gavis::MappingContext mc;
    mc.vmf = gavis::VmfParams(kappa);
    mc.field_degree = degree;
    mc.raster = make_rc(rc);
    mc.uncertainty = make_uc(u);
    mc.density.rho = rho;
    mc.density.eta = eta;
    mc.density.eps_v = eps_v;
    mc.density.seed = dseed;
    mc.density_enabled = density_enabled != 0;
    const gavis::PlannerConfig p = make_pc(pc);
    const gavis::MappingLog log =
        gavis::run_active_mapping(sc, make_occluders(rects, n_rects, density), t, p, mc, threads);
    for (size_t k = 0; k < log.steps.size(); ++k) {
      chosen[k] = log.steps[k].chosen_index;
      score[k] = log.steps[k].score;
      coverage[k] = log.steps[k].vis_coverage;
      std::memcpy(all_scores + k * (size_t)p.num_candidates, log.steps[k].scores.data(),
                  sizeof(double) * log.steps[k].scores.size());
    }
  });
}

// render_entropy_core (uncertainty.hpp:124-238) with per-particle visibilities,
// optional sh_propagation coefficient variances [N][3][(Lv+1)^2] (coeff_var NULL:
// the constant provider), entropy / w0 / depth per pixel, and the per-pixel
// mixtures in gor_render_mixtures's layout (offsets[P+1] always; components and
// the per-pixel prior / residual T / H when comps is non-NULL, capacity cap).
int gref_render_entropy_core(const gor_scene* s, const gor_camera* cam, const gor_raster* rc, const gor_unc* u,
                             const double* vis_by_particle, const double* coeff_var, int var_degree, int threads,
                             double* H, double* w0, double* depth, int64_t* offsets, gor_mixture_component* comps,
                             int64_t cap, double* prior, double* resid, double* Hm) {
  return guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const gavis::CameraView cv = make_cam(cam);
    const gavis::RasterConfig r = make_rc(rc);
    gavis::UncertaintyConfig uc = make_uc(u);
    std::vector<std::array<std::vector<double>, 3>> var;
    if (coeff_var) {
      const size_t nb = (size_t)(var_degree + 1) * (var_degree + 1);
      var.resize(sc.particles.size());
      for (size_t i = 0; i < var.size(); ++i)
        for (int c = 0; c < 3; ++c) var[i][c].assign(coeff_var + (i * 3 + c) * nb, coeff_var + (i * 3 + c + 1) * nb);
      uc.variance_provider = gavis::VarianceProvider::kShPropagation;
      uc.coeff_variances = &var;
    }
    const gavis::ProjectedView pv = gavis::project_scene(sc, cv, r.dilation);
    std::vector<double> sv(pv.splats.size());
    for (size_t k = 0; k < sv.size(); ++k) sv[k] = vis_by_particle[pv.splats[k].particle_index];
    std::vector<double> d;
    std::vector<gavis::PixelMixture> mix;
    const gavis::EntropyMap m = gavis::render_entropy_core(sc, pv, sv, cv, r, uc, threads, &d,
                                                           offsets ? &mix : nullptr);
    if (H) std::memcpy(H, m.entropy.data(), sizeof(double) * m.entropy.size());
    if (w0) std::memcpy(w0, m.invisible_mass.data(), sizeof(double) * m.invisible_mass.size());
    if (depth) std::memcpy(depth, d.data(), sizeof(double) * d.size());
    if (offsets) {
      int64_t k = 0;
      for (size_t p = 0; p < mix.size(); ++p) {
        offsets[p] = k;
        if (comps) {
          for (const auto& c : mix[p].components) {
            if (k >= cap) throw gavis::InvariantError("render_entropy_core: component capacity too small");
            gor_mixture_component& o = comps[k];
            o.weight = c.weight;
            o.vis = c.vis;
            for (int j = 0; j < 3; ++j) {
              o.mean[j] = c.mean[j];
              o.var[j] = c.var[j];
            }
            ++k;
          }
          if (prior) prior[p] = mix[p].prior_weight;
          if (resid) resid[p] = mix[p].residual_transmittance;
          if (Hm) Hm[p] = mix[p].entropy;
        } else {
          k += (int64_t)mix[p].components.size();
        }
      }
      offsets[mix.size()] = k;
    }
  });
}

// project_scene (raster.hpp:114-130) -> splats sorted by (depth, index), count;
// splat_binning (raster.hpp:145-164) of them -> CSR tile lists (entries NULL: size)
int64_t gref_project_and_bin(const gor_scene* s, const gor_camera* cam, double dilation, int tile_size,
                             gor_splat* splats, int64_t* tile_offsets, int32_t* entries) {
  int64_t total = -1;
  const int st = guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const gavis::CameraView cv = make_cam(cam);
    const gavis::ProjectedView pv = gavis::project_scene(sc, cv, dilation);
    for (size_t k = 0; k < pv.splats.size(); ++k) {
      const gavis::ImageSpaceSplat& a = pv.splats[k];
      gor_splat& o = splats[k];
      o.particle_index = a.particle_index;
      o._pad = 0;
      o.mean_x = a.mean.x();
      o.mean_y = a.mean.y();
      o.conic_a = a.conic_a;
      o.conic_b = a.conic_b;
      o.conic_c = a.conic_c;
      o.depth = a.depth;
      o.radius = a.radius;
      o.opacity = a.opacity;
    }
    const gavis::SplatBinning b = gavis::splat_binning(pv.splats, cv.width, cv.height, tile_size);
    int64_t k = 0;
    for (size_t t = 0; t < b.tiles.size(); ++t) {
      tile_offsets[t] = k;
      for (int e : b.tiles[t]) {
        if (entries) entries[k] = e;
        ++k;
      }
    }
    tile_offsets[b.tiles.size()] = k;
    total = (int64_t)pv.splats.size();
  });
  return st == 0 ? total : -st;
}

// query_view (vfield.hpp:121-134) -> the non-culled particle indices and their
// visibilities; returns the count
int64_t gref_query_view(const gor_scene* s, const double* gamma, int degree, int num_views, const gor_camera* cam,
                        double dilation, int32_t* idx, double* vis) {
  int64_t n = -1;
  const int st = guarded([&] {
    const gavis::Scene sc = make_scene(s);
    const gavis::VisibilityField f = make_field(sc, gamma, degree, num_views);
    const gavis::ViewQuery q = gavis::query_view(f, sc, make_cam(cam), dilation);
    for (size_t k = 0; k < q.particle_indices.size(); ++k) {
      idx[k] = q.particle_indices[k];
      vis[k] = q.visibilities[k];
    }
    n = (int64_t)q.particle_indices.size();
  });
  return st == 0 ? n : -st;
}

}  // extern "C"
