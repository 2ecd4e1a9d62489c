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

}  // extern "C"
