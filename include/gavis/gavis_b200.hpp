// gavis_b200.hpp -- header-only C++ front-end with the reference's signatures.
//
// A caller of the GAVIS reference (R/ = /root/reference/proj/include/gavis/)
// swaps its hot-path calls for these, keeping argument meaning and error
// behaviour:
//   construct_field          vfield.hpp:68-70
//   accumulate_view          vfield.hpp:38-40
//   single_view_visibility   raster.hpp:237-238
//   query_visibility         vfield.hpp:96-97
//   query_view               vfield.hpp:121-122
//   rasterize                raster.hpp:175-176
//   render_entropy           uncertainty.hpp:242-246
//   image_entropy            uncertainty.hpp:264-265
//   select_nbv               planner.hpp:117-120
// Eigen is not required: Vec3 / Mat3 / Quat are small PODs with the same
// element order (Quat = (w, x, y, z), Mat3 row-major accessors m(r, c)).
// ParameterError / InvariantError are thrown where the reference throws them;
// device failures throw DeviceError. The `threads` arguments are accepted for
// source compatibility; the work runs on the GPU of the default context
// (device 0, or set_default_device()).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../gavis_b200.h"

namespace gavis_b200 {

inline constexpr double kPi = 3.14159265358979323846;
inline constexpr double kY00 = 0.28209479177387814;

class ParameterError : public std::runtime_error {
 public:
  explicit ParameterError(const std::string& m) : std::runtime_error(m) {}
};
class InvariantError : public std::logic_error {
 public:
  explicit InvariantError(const std::string& m) : std::logic_error(m) {}
};
class OracleError : public std::runtime_error {
 public:
  explicit OracleError(const std::string& m) : std::runtime_error(m) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

inline void check(gavis_status s) {
  if (s == GAVIS_OK) return;
  const std::string msg = gavis_last_error();
  switch (s) {
    case GAVIS_ERR_PARAMETER: throw ParameterError(msg);
    case GAVIS_ERR_INVARIANT: throw InvariantError(msg);
    case GAVIS_ERR_ORACLE: throw OracleError(msg);
    default: throw DeviceError(msg);
  }
}

struct Vec3 {
  double v[3] = {0, 0, 0};
  Vec3() = default;
  Vec3(double x, double y, double z) : v{x, y, z} {}
  double x() const { return v[0]; }
  double y() const { return v[1]; }
  double z() const { return v[2]; }
  double& operator[](int i) { return v[i]; }
  double operator[](int i) const { return v[i]; }
};

struct Mat3 {
  double m[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};  // row-major
  double& operator()(int r, int c) { return m[r * 3 + c]; }
  double operator()(int r, int c) const { return m[r * 3 + c]; }
};

struct Quat {
  double w = 1, x = 0, y = 0, z = 0;  // Eigen ctor order (w, x, y, z)
};

// model.hpp:34-46
struct GaussianParticle {
  Vec3 position;
  Quat rotation;
  Vec3 scale{1, 1, 1};
  double opacity = 0.0;
  std::array<std::vector<double>, 3> color_sh;
  bool is_virtual = false;
};

struct Bounds {
  Vec3 min, max;
};

// model.hpp:130-138
struct Scene {
  int color_degree = 0;
  Bounds bounds;
  std::vector<GaussianParticle> particles;
};

// model.hpp:66-105
struct CameraView {
  Mat3 rotation;  // columns: right, down, forward
  Vec3 position;
  int width = 128, height = 128;
  double fov_h = kPi / 2.0, fov_v = kPi / 2.0, near = 0.05;
};

struct Trajectory {
  std::vector<CameraView> views;
};

// raster.hpp:21-35
struct RasterConfig {
  int tile_size = 16;
  double transmittance_cutoff = 1e-4;
  double dilation = 0.3;
  double alpha_clamp_max = 0.99;
};

// sh.hpp:121-129
struct VmfParams {
  double kappa = 1.0;
  double zeta = std::exp(-1.0);
  VmfParams() = default;
  explicit VmfParams(double k) : kappa(k), zeta(std::exp(-k)) {
    if (!(k >= 0.0 && k <= 50.0)) throw ParameterError("vmf kappa must lie in [0, 50]");
  }
};

// uncertainty.hpp:21-22
enum class VarianceProvider { kConstant, kShPropagation };
enum class CorrelationMode { kNone, kHook };

// uncertainty.hpp:24-52
struct UncertaintyConfig {
  double beta = 0.5;
  double prior_opacity = 0.15;           // o_0
  Mat3 prior_cov;                        // Q_0 (identity)
  double color_sigma = 0.1;              // Q_c = sigma^2 I under kConstant
  VarianceProvider variance_provider = VarianceProvider::kConstant;
  CorrelationMode correlation = CorrelationMode::kNone;
  double correlation_lambda = 1.0;
  // Only mixture dumps read the prior mean (uncertainty.hpp:32-34).
  Vec3 prior_mean = Vec3(0.5, 0.5, 0.5);
  // Per-particle per-channel SH coefficient variances for kShPropagation
  // (uncertainty.hpp:35-37): [N][3][(Lv+1)^2], Lv <= 4 on the device.
  const std::vector<std::array<std::vector<double>, 3>>* coeff_variances = nullptr;
};

// vfield.hpp:21-33
struct VisibilityField {
  int degree = 2;
  VmfParams vmf;
  int num_views = 0;
  std::size_t num_particles = 0;
  std::vector<double> gamma;
  std::vector<uint8_t> virtual_mask;
  int basis_size() const { return (degree + 1) * (degree + 1); }
  const double* coeffs(std::size_t p) const { return gamma.data() + p * basis_size(); }
};

struct ViewQuery {
  std::vector<int> particle_indices;
  std::vector<double> visibilities;
};

struct EntropyMap {
  int width = 0, height = 0;
  std::vector<double> entropy;
  std::vector<double> invisible_mass;
};

// uncertainty.hpp:90-102
struct PixelMixtureComponent {
  double weight = 0.0;  // w* = alpha* T
  double vis = 0.0;     // particle visibility v
  Vec3 mean{};
  Vec3 var{};           // diagonal of Q_c
};

struct PixelMixture {
  int x = 0, y = 0;
  double prior_weight = 0.0;            // w0
  double residual_transmittance = 0.0;  // T after the loop
  double entropy = 0.0;
  std::vector<PixelMixtureComponent> components;
};

struct RenderOutput {
  int width = 0, height = 0;
  std::vector<double> color, depth, transmittance;
};

struct NbvResult {
  int best_index = -1;
  std::vector<double> scores;
};

namespace detail {

struct CtxHolder {
  gavis_ctx* ctx = nullptr;
  int device = 0;
  ~CtxHolder() {
    if (ctx) gavis_ctx_destroy(ctx);
  }
  gavis_ctx* get() {
    if (!ctx) check(gavis_ctx_create(device, nullptr, &ctx));
    return ctx;
  }
};

inline CtxHolder& holder() {
  static CtxHolder h;
  return h;
}

inline gavis_camera cam_c(const CameraView& c) {
  gavis_camera g{};
  for (int i = 0; i < 9; ++i) g.rotation[i] = c.rotation.m[i];
  for (int i = 0; i < 3; ++i) g.position[i] = c.position[i];
  g.width = c.width;
  g.height = c.height;
  g.fov_h = c.fov_h;
  g.fov_v = c.fov_v;
  g.near_plane = c.near;
  return g;
}

inline gavis_raster_config rc_c(const RasterConfig& r) {
  return gavis_raster_config{r.tile_size, 0, r.transmittance_cutoff, r.dilation, r.alpha_clamp_max};
}

inline gavis_uncertainty_config uc_c(const UncertaintyConfig& u) {
  gavis_uncertainty_config g{};
  g.beta = u.beta;
  g.prior_opacity = u.prior_opacity;
  g.color_sigma = u.color_sigma;
  for (int i = 0; i < 9; ++i) g.prior_cov[i] = u.prior_cov.m[i];
  g.variance_provider = u.variance_provider == VarianceProvider::kShPropagation ? 1 : 0;
  g.correlation = u.correlation == CorrelationMode::kHook ? 1 : 0;
  g.correlation_lambda = u.correlation_lambda;
  return g;
}

// Scene (AoS, double) -> device scene (fp32 SoA). Owns the device handle.
struct DeviceScene {
  gavis_scene* h = nullptr;
  ~DeviceScene() {
    if (h) gavis_scene_destroy(h);
  }
};

inline std::unique_ptr<DeviceScene> upload(const Scene& s) {
  const std::size_t n = s.particles.size();
  const int nb = (s.color_degree + 1) * (s.color_degree + 1);
  std::vector<float> pos(3 * n), rot(4 * n), scl(3 * n), op(n), col(3 * nb * n, 0.f);
  std::vector<uint8_t> virt(n);
  for (std::size_t i = 0; i < n; ++i) {
    const GaussianParticle& p = s.particles[i];
    for (int k = 0; k < 3; ++k) {
      pos[3 * i + k] = (float)p.position[k];
      scl[3 * i + k] = (float)p.scale[k];
      const std::size_t cnt = std::min<std::size_t>(nb, p.color_sh[k].size());
      for (std::size_t j = 0; j < cnt; ++j) col[(3 * i + k) * nb + j] = (float)p.color_sh[k][j];
    }
    rot[4 * i] = (float)p.rotation.w;
    rot[4 * i + 1] = (float)p.rotation.x;
    rot[4 * i + 2] = (float)p.rotation.y;
    rot[4 * i + 3] = (float)p.rotation.z;
    op[i] = (float)p.opacity;
    virt[i] = p.is_virtual ? 1 : 0;
  }
  gavis_scene_desc d{};
  d.num_particles = (int64_t)n;
  d.color_degree = s.color_degree;
  d.positions = pos.data();
  d.rotations = rot.data();
  d.scales = scl.data();
  d.opacities = op.data();
  d.colors = col.data();
  d.is_virtual = virt.data();
  auto ds = std::make_unique<DeviceScene>();
  check(gavis_scene_upload(holder().get(), &d, &ds->h));
  return ds;
}

// UncertaintyConfig::coeff_variances -> the device scene (kShPropagation).
inline void attach_variances(const UncertaintyConfig& uc, gavis_scene* s, std::size_t n) {
  if (uc.variance_provider != VarianceProvider::kShPropagation) return;
  if (uc.coeff_variances == nullptr)
    throw ParameterError("variance_provider sh_propagation requires coeff_variances");
  const auto& cv = *uc.coeff_variances;
  if (cv.size() != n) throw ParameterError("coeff_variances: one entry per particle");
  const std::size_t nb = n ? cv[0][0].size() : 1;
  int deg = 0;
  while ((std::size_t)((deg + 1) * (deg + 1)) < nb) ++deg;
  if ((std::size_t)((deg + 1) * (deg + 1)) != nb)
    throw ParameterError("coeff_variances: channel rows must hold complete SH bands");
  std::vector<float> flat(n * 3 * nb);
  for (std::size_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      if (cv[i][c].size() != nb) throw ParameterError("coeff_variances: ragged channel rows");
      for (std::size_t k = 0; k < nb; ++k) flat[(i * 3 + c) * nb + k] = (float)cv[i][c][k];
    }
  check(gavis_scene_set_coeff_variances(holder().get(), s, flat.empty() ? nullptr : flat.data(), deg));
}

struct DeviceField {
  gavis_field* h = nullptr;
  ~DeviceField() {
    if (h) gavis_vf_destroy(h);
  }
};

inline std::unique_ptr<DeviceField> upload_field(const VisibilityField& f, const DeviceScene& s) {
  auto df = std::make_unique<DeviceField>();
  check(gavis_vf_upload(holder().get(), s.h, f.vmf.kappa, f.degree, f.num_views,
                        f.gamma.empty() ? nullptr : f.gamma.data(), &df->h));
  return df;
}

inline std::vector<uint8_t> virtual_mask(const Scene& s) {
  std::vector<uint8_t> m(s.particles.size());
  for (std::size_t i = 0; i < m.size(); ++i) m[i] = s.particles[i].is_virtual ? 1 : 0;
  return m;
}

}  // namespace detail

inline void set_default_device(int device) { detail::holder().device = device; }

// Arithmetic of the UA render (gavis_ctx_set_precision): the fp64 blend (default,
// the reference's arithmetic) or the certified fp32 blend (contributor counts and
// the selected view equal the fp64 reference's, images to ~1e-6).
inline void set_exact_precision(bool exact) {
  check(gavis_ctx_set_precision(detail::holder().get(),
                                exact ? GAVIS_PRECISION_EXACT : GAVIS_PRECISION_CERTIFIED));
}

// vfield.hpp:68-92
inline VisibilityField construct_field(const Scene& scene, const Trajectory& trajectory,
                                       const VmfParams& vmf, int degree,
                                       const RasterConfig& rc = {}, int /*threads*/ = 1) {
  auto ds = detail::upload(scene);
  std::vector<gavis_camera> cams;
  for (const auto& v : trajectory.views) cams.push_back(detail::cam_c(v));
  const gavis_raster_config r = detail::rc_c(rc);
  gavis_field* f = nullptr;
  check(gavis_vf_construct(detail::holder().get(), ds->h, cams.data(), (int32_t)cams.size(),
                           vmf.kappa, degree, &r, &f));
  detail::DeviceField guard{f};
  VisibilityField out;
  out.degree = degree;
  out.vmf = vmf;
  out.num_particles = scene.particles.size();
  out.gamma.resize(out.num_particles * out.basis_size());
  int32_t nv = 0;
  check(gavis_vf_download(f, out.gamma.empty() ? nullptr : out.gamma.data(), &nv, nullptr));
  out.num_views = nv;
  out.virtual_mask = detail::virtual_mask(scene);
  return out;
}

// vfield.hpp:38-63
inline void accumulate_view(VisibilityField& field, const Scene& scene, const CameraView& view,
                            const std::vector<double>& visibility, int /*threads*/ = 1) {
  if (field.num_particles != scene.particles.size())
    throw InvariantError("accumulate_view: field/scene particle count mismatch");
  auto ds = detail::upload(scene);
  auto df = detail::upload_field(field, *ds);
  const gavis_camera c = detail::cam_c(view);
  check(gavis_vf_accumulate_visibility(detail::holder().get(), df->h, ds->h, &c,
                                       visibility.empty() ? nullptr : visibility.data()));
  int32_t nv = 0;
  check(gavis_vf_download(df->h, field.gamma.empty() ? nullptr : field.gamma.data(), &nv, nullptr));
  field.num_views = nv;
}

// raster.hpp:237-290
inline std::vector<double> single_view_visibility(const Scene& scene, const CameraView& cam,
                                                  const RasterConfig& rc, int /*threads*/ = 1) {
  auto ds = detail::upload(scene);
  const gavis_camera c = detail::cam_c(cam);
  const gavis_raster_config r = detail::rc_c(rc);
  std::vector<double> v(scene.particles.size());
  check(gavis_single_view_visibility(detail::holder().get(), ds->h, &c, &r,
                                     v.empty() ? nullptr : v.data(), nullptr, nullptr));
  return v;
}

// vfield.hpp:96-112 (particle index and a unit direction)
inline double query_visibility(const VisibilityField& field, std::size_t particle_index,
                               const Vec3& d) {
  if (particle_index >= field.num_particles)
    throw ParameterError("query: particle index out of range");
  if (field.virtual_mask.size() == field.num_particles && field.virtual_mask[particle_index])
    return 0.0;
  // single-row field on the device: one particle, same coefficients
  Scene one;
  one.particles.resize(1);
  auto ds = detail::upload(one);
  VisibilityField row;
  row.degree = field.degree;
  row.vmf = field.vmf;
  row.num_views = field.num_views;
  row.num_particles = 1;
  row.gamma.assign(field.coeffs(particle_index), field.coeffs(particle_index) + field.basis_size());
  auto df = detail::upload_field(row, *ds);
  const int64_t idx = 0;
  double out = 0.0;
  check(gavis_vf_query(detail::holder().get(), df->h, &idx, d.v, 1, &out));
  return out;
}

// vfield.hpp:121-134
inline ViewQuery query_view(const VisibilityField& field, const Scene& scene,
                            const CameraView& camera, double dilation = 0.3) {
  if (field.num_particles != scene.particles.size())
    throw ParameterError("query_view: field/scene particle count mismatch");
  auto ds = detail::upload(scene);
  auto df = detail::upload_field(field, *ds);
  const gavis_camera c = detail::cam_c(camera);
  std::vector<int32_t> idx(scene.particles.size());
  std::vector<double> vis(scene.particles.size());
  int64_t n = 0;
  check(gavis_vf_query_view(detail::holder().get(), df->h, ds->h, &c, dilation,
                            idx.empty() ? nullptr : idx.data(), vis.empty() ? nullptr : vis.data(), &n));
  ViewQuery q;
  q.particle_indices.assign(idx.begin(), idx.begin() + n);
  q.visibilities.assign(vis.begin(), vis.begin() + n);
  return q;
}

// raster.hpp:175-231
inline RenderOutput rasterize(const Scene& scene, const CameraView& cam, const RasterConfig& rc,
                              int /*threads*/ = 1) {
  auto ds = detail::upload(scene);
  const gavis_camera c = detail::cam_c(cam);
  const gavis_raster_config r = detail::rc_c(rc);
  const gavis_uncertainty_config u = detail::uc_c(UncertaintyConfig{});
  RenderOutput out;
  out.width = cam.width;
  out.height = cam.height;
  const std::size_t P = (std::size_t)cam.width * cam.height;
  out.color.resize(3 * P);
  out.depth.resize(P);
  out.transmittance.resize(P);
  gavis_render_outputs o{};
  o.rgb = out.color.data();
  o.depth = out.depth.data();
  o.transmittance = out.transmittance.data();
  check(gavis_ua_render(detail::holder().get(), ds->h, nullptr, nullptr, &c, 1, &r, &u, &o));
  return out;
}

// uncertainty.hpp:242-260
inline EntropyMap render_entropy(const Scene& scene, const VisibilityField& field,
                                 const CameraView& cam, const RasterConfig& rc,
                                 const UncertaintyConfig& uc, int /*threads*/ = 1,
                                 std::vector<double>* depth_out = nullptr,
                                 std::vector<PixelMixture>* mixtures_out = nullptr) {
  if (field.num_particles != scene.particles.size())
    throw ParameterError("render_entropy: field was built for a different scene");
  auto ds = detail::upload(scene);
  detail::attach_variances(uc, ds->h, scene.particles.size());
  auto df = detail::upload_field(field, *ds);
  const gavis_camera c = detail::cam_c(cam);
  const gavis_raster_config r = detail::rc_c(rc);
  const gavis_uncertainty_config u = detail::uc_c(uc);
  EntropyMap m;
  m.width = cam.width;
  m.height = cam.height;
  const std::size_t P = (std::size_t)cam.width * cam.height;
  m.entropy.resize(P);
  m.invisible_mass.resize(P);
  if (depth_out) depth_out->resize(P);
  gavis_render_outputs o{};
  o.entropy = m.entropy.data();
  o.invisible_mass = m.invisible_mass.data();
  o.entropy_depth = depth_out ? depth_out->data() : nullptr;
  check(gavis_ua_render(detail::holder().get(), ds->h, df->h, nullptr, &c, 1, &r, &u, &o));
  if (mixtures_out) {
    // uncertainty.hpp:207-230: per-pixel components (exact fp64 track on the device)
    std::vector<int64_t> off(P + 1);
    std::vector<double> prior(P), resid(P), ent(P);
    check(gavis_ua_mixtures(detail::holder().get(), ds->h, df->h, nullptr, &c, &r, &u, off.data(),
                            nullptr, 0, prior.data(), resid.data(), ent.data()));
    std::vector<gavis_mixture_component> comp((std::size_t)off[P]);
    if (!comp.empty())
      check(gavis_ua_mixtures(detail::holder().get(), ds->h, df->h, nullptr, &c, &r, &u, off.data(),
                              comp.data(), (int64_t)comp.size(), nullptr, nullptr, nullptr));
    mixtures_out->assign(P, PixelMixture{});
    for (std::size_t p = 0; p < P; ++p) {
      PixelMixture& mx = (*mixtures_out)[p];
      mx.x = (int)(p % (std::size_t)cam.width);
      mx.y = (int)(p / (std::size_t)cam.width);
      mx.prior_weight = prior[p];
      mx.residual_transmittance = resid[p];
      mx.entropy = ent[p];
      for (int64_t k = off[p]; k < off[p + 1]; ++k) {
        const gavis_mixture_component& g = comp[(std::size_t)k];
        mx.components.push_back({g.weight, g.vis, Vec3{g.mean[0], g.mean[1], g.mean[2]},
                                 Vec3{g.var[0], g.var[1], g.var[2]}});
      }
    }
  }
  return m;
}

// uncertainty.hpp:264-278: correlation none -> plain sum in pixel order; hook ->
// sum of H - H exp(-d / lambda) with d the entropy depth (a host fold of the
// maps the caller already holds; select_nbv folds on the device).
inline double image_entropy(const EntropyMap& map, const std::vector<double>& depth,
                            const UncertaintyConfig& uc) {
  if (depth.size() != map.entropy.size())
    throw ParameterError("image_entropy: depth map shape differs from the entropy map");
  double sum = 0.0;
  if (uc.correlation == CorrelationMode::kNone) {
    for (double h : map.entropy) sum += h;
    return sum;
  }
  for (std::size_t i = 0; i < map.entropy.size(); ++i) {
    const double h = map.entropy[i];
    sum += h - h * std::exp(-depth[i] / uc.correlation_lambda);
  }
  return sum;
}

// planner.hpp:117-137
inline NbvResult select_nbv(const Scene& scene_aug, const VisibilityField& field,
                            const std::vector<CameraView>& candidates, const RasterConfig& rc,
                            const UncertaintyConfig& uc, int /*threads*/ = 1) {
  if (candidates.empty()) throw ParameterError("select_nbv: candidate list must be nonempty");
  auto ds = detail::upload(scene_aug);
  detail::attach_variances(uc, ds->h, scene_aug.particles.size());
  auto df = detail::upload_field(field, *ds);
  std::vector<gavis_camera> cams;
  for (const auto& v : candidates) cams.push_back(detail::cam_c(v));
  const gavis_raster_config r = detail::rc_c(rc);
  const gavis_uncertainty_config u = detail::uc_c(uc);
  NbvResult res;
  res.scores.resize(candidates.size());
  int32_t best = -1;
  check(gavis_select_nbv(detail::holder().get(), ds->h, df->h, cams.data(), (int32_t)cams.size(),
                         &r, &u, 0, res.scores.data(), &best));
  res.best_index = best;
  return res;
}

// model.hpp:107-128
inline CameraView make_lookat(const Vec3& position, const Vec3& target, const Vec3& up = Vec3(0, 0, 1),
                              int width = 128, int height = 128, double fov_h = kPi / 2.0,
                              double fov_v = kPi / 2.0) {
  auto sub = [](const Vec3& a, const Vec3& b) { return Vec3(a[0] - b[0], a[1] - b[1], a[2] - b[2]); };
  auto cross = [](const Vec3& a, const Vec3& b) {
    return Vec3(a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]);
  };
  auto norm = [](const Vec3& a) { return std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]); };
  auto unit = [&](const Vec3& a) {
    const double n = norm(a);
    return Vec3(a[0] / n, a[1] / n, a[2] / n);
  };
  Vec3 forward = sub(target, position);
  if (!(norm(forward) > 1e-12)) throw ParameterError("lookat target coincides with position");
  forward = unit(forward);
  Vec3 right = cross(forward, up);
  if (norm(right) < 1e-9) right = cross(forward, Vec3(1, 0, 0));
  right = unit(right);
  const Vec3 down = cross(forward, right);
  CameraView v;
  for (int r = 0; r < 3; ++r) {
    v.rotation(r, 0) = right[r];
    v.rotation(r, 1) = down[r];
    v.rotation(r, 2) = forward[r];
  }
  v.position = position;
  v.width = width;
  v.height = height;
  v.fov_h = fov_h;
  v.fov_v = fov_v;
  return v;
}

// ---- density control (vfield.hpp:136-199) ---------------------------------
struct DensityControlConfig {
  double rho = 100.0, eta = 0.5, eps_v = 0.95;
  uint64_t seed = 0;
};

inline double virtual_particle_scale(const DensityControlConfig& cfg) {
  return std::cbrt(3.0 * (1.0 + cfg.eta) / (4.0 * kPi * cfg.rho));
}

namespace detail {
inline uint64_t mix64(uint64_t x) {  // rng.hpp:18-28
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
inline gavis_density_config dc_c(const DensityControlConfig& d) {
  return gavis_density_config{d.rho, d.eta, d.eps_v, d.seed};
}
inline CameraView cam_from_c(const gavis_camera& g) {
  CameraView c;
  for (int i = 0; i < 9; ++i) c.rotation.m[i] = g.rotation[i];
  c.position = Vec3(g.position[0], g.position[1], g.position[2]);
  c.width = g.width;
  c.height = g.height;
  c.fov_h = g.fov_h;
  c.fov_v = g.fov_v;
  c.near = g.near_plane;
  return c;
}
}  // namespace detail

inline uint64_t derive_seed(uint64_t seed, uint64_t stream) {
  return detail::mix64(seed ^ detail::mix64(stream + 0x632be59bd9b4e019ull));
}

// The device decides which probes survive (isotropic multi-view visibility on
// the VF kernels); the returned host scene appends them exactly as the
// reference does (double positions bounds.min + extent * u, scale s, o = 0).
inline Scene density_control(const Scene& scene, const Trajectory& trajectory,
                             const DensityControlConfig& cfg, const RasterConfig& rc = {},
                             int /*threads*/ = 1) {
  auto ds = detail::upload(scene);
  std::vector<gavis_camera> views;
  for (const auto& v : trajectory.views) views.push_back(detail::cam_c(v));
  const double bmin[3] = {scene.bounds.min[0], scene.bounds.min[1], scene.bounds.min[2]};
  const double bmax[3] = {scene.bounds.max[0], scene.bounds.max[1], scene.bounds.max[2]};
  const double ext[3] = {bmax[0] - bmin[0], bmax[1] - bmin[1], bmax[2] - bmin[2]};
  const double vol = ext[0] * ext[1] * ext[2];
  const std::size_t cap = vol > 0.0 && cfg.rho > 0.0 ? (std::size_t)std::floor(cfg.rho * vol) : 0;
  std::vector<int64_t> kept(std::max<std::size_t>(1, cap));
  int64_t n_kept = 0;
  gavis_scene* aug = nullptr;
  const gavis_density_config d = detail::dc_c(cfg);
  const gavis_raster_config r = detail::rc_c(rc);
  check(gavis_density_control(detail::holder().get(), ds->h, bmin, bmax, views.data(),
                              (int32_t)views.size(), &d, &r, &aug, &n_kept, kept.data(),
                              (int64_t)kept.size()));
  gavis_scene_destroy(aug);
  Scene out = scene;
  const double s = virtual_particle_scale(cfg);
  const int nb = (scene.color_degree + 1) * (scene.color_degree + 1);
  for (int64_t i = 0; i < n_kept; ++i) {
    uint64_t st = derive_seed(cfg.seed, (uint64_t)kept[i]);
    double u[3];
    for (int k = 0; k < 3; ++k) {
      st += 0x9e3779b97f4a7c15ull;
      u[k] = (double)(detail::mix64(st - 0x9e3779b97f4a7c15ull) >> 11) * 0x1.0p-53;
    }
    GaussianParticle vp;
    vp.position = Vec3(bmin[0] + ext[0] * u[0], bmin[1] + ext[1] * u[1], bmin[2] + ext[2] * u[2]);
    vp.scale = Vec3(s, s, s);
    vp.opacity = 0.0;
    vp.is_virtual = true;
    for (int c = 0; c < 3; ++c) vp.color_sh[c].assign(nb, 0.0);
    out.particles.push_back(vp);
  }
  return out;
}

// ---- planner (planner.hpp) --------------------------------------------------
enum class PoseMode { kSe3, kSe2 };

struct PlannerConfig {  // planner.hpp:24-42
  PoseMode mode = PoseMode::kSe3;
  int num_candidates = 128;
  double se2_height = 1.5;
  int steps = 10;
  uint64_t seed = 0;
  bool look_inward = true;
  double clearance = 0.1;
  int cam_width = 128, cam_height = 128;
  double fov_h = kPi / 2.0, fov_v = kPi / 2.0;
  double cam_near = 0.05;
};

struct OccluderRect {  // model.hpp:141-150
  Vec3 corner = Vec3(0, 0, 0), edge_u = Vec3(1, 0, 0), edge_v = Vec3(0, 1, 0);
  bool opaque = true;
};

struct OccluderSet {  // model.hpp:152-155
  std::vector<OccluderRect> rectangles;
  double sample_density = 64.0;
};

struct MappingContext {  // planner.hpp:255-262
  VmfParams vmf;
  int field_degree = 2;
  RasterConfig raster;
  UncertaintyConfig uncertainty;
  DensityControlConfig density;
  bool density_enabled = true;
};

struct MappingStep {  // planner.hpp:264-270
  std::vector<double> scores;
  int chosen_index = -1;
  double score = 0.0, vis_coverage = 0.0, mean_entropy = 0.0;
};

struct MappingLog {  // planner.hpp:272-275
  Trajectory chosen_views;
  std::vector<MappingStep> steps;
};

namespace detail {
inline std::vector<gavis_occluder_rect> rects_c(const OccluderSet& o) {
  std::vector<gavis_occluder_rect> out;
  for (const auto& r : o.rectangles) {
    gavis_occluder_rect g{};
    for (int k = 0; k < 3; ++k) {
      g.corner[k] = r.corner[k];
      g.edge_u[k] = r.edge_u[k];
      g.edge_v[k] = r.edge_v[k];
    }
    g.opaque = r.opaque ? 1 : 0;
    out.push_back(g);
  }
  return out;
}
inline gavis_planner_config pc_c(const PlannerConfig& p) {
  gavis_planner_config g{};
  g.mode = p.mode == PoseMode::kSe2 ? 1 : 0;
  g.num_candidates = p.num_candidates;
  g.se2_height = p.se2_height;
  g.steps = p.steps;
  g.look_inward = p.look_inward ? 1 : 0;
  g.seed = p.seed;
  g.clearance = p.clearance;
  g.cam_width = p.cam_width;
  g.cam_height = p.cam_height;
  g.fov_h = p.fov_h;
  g.fov_v = p.fov_v;
  g.cam_near = p.cam_near;
  return g;
}
}  // namespace detail

// planner.hpp:56-107 (host code in the library; no device needed)
inline std::vector<CameraView> sample_candidates(const Bounds& bounds, const OccluderSet& occluders,
                                                 const PlannerConfig& pc, uint64_t step_seed) {
  const auto rects = detail::rects_c(occluders);
  const gavis_planner_config g = detail::pc_c(pc);
  std::vector<gavis_camera> out(std::max(1, pc.num_candidates));
  const double bmin[3] = {bounds.min[0], bounds.min[1], bounds.min[2]};
  const double bmax[3] = {bounds.max[0], bounds.max[1], bounds.max[2]};
  check(gavis_sample_candidates(bmin, bmax, rects.data(), (int32_t)rects.size(), &g, step_seed,
                                out.data()));
  std::vector<CameraView> views;
  for (int i = 0; i < pc.num_candidates; ++i) views.push_back(detail::cam_from_c(out[i]));
  return views;
}

// planner.hpp:155-184
inline double vis_coverage(const OccluderSet& occluders, const Trajectory& trajectory) {
  const auto rects = detail::rects_c(occluders);
  std::vector<gavis_camera> views;
  for (const auto& v : trajectory.views) views.push_back(detail::cam_c(v));
  double cov = 0.0;
  check(gavis_vis_coverage(rects.data(), (int32_t)rects.size(), occluders.sample_density,
                           views.data(), (int32_t)views.size(), &cov));
  return cov;
}

// planner.hpp:284-316
inline MappingLog run_active_mapping(const Scene& scene, const OccluderSet& occluders,
                                     const Trajectory& init, const PlannerConfig& pc,
                                     const MappingContext& ctx, int /*threads*/ = 1) {
  auto ds = detail::upload(scene);
  detail::attach_variances(ctx.uncertainty, ds->h, scene.particles.size());
  const auto rects = detail::rects_c(occluders);
  const gavis_planner_config g = detail::pc_c(pc);
  gavis_mapping_config mc{};
  mc.kappa = ctx.vmf.kappa;
  mc.field_degree = ctx.field_degree;
  mc.density_enabled = ctx.density_enabled ? 1 : 0;
  mc.raster = detail::rc_c(ctx.raster);
  mc.uncertainty = detail::uc_c(ctx.uncertainty);
  mc.density = detail::dc_c(ctx.density);
  std::vector<gavis_camera> init_c;
  for (const auto& v : init.views) init_c.push_back(detail::cam_c(v));
  const int steps = std::max(0, pc.steps), nc = std::max(1, pc.num_candidates);
  std::vector<gavis_camera> chosen(std::max(1, steps));
  std::vector<int32_t> idx(std::max(1, steps));
  std::vector<double> score(std::max(1, steps)), all((size_t)std::max(1, steps) * nc),
      cov(std::max(1, steps)), ment(std::max(1, steps));
  const double bmin[3] = {scene.bounds.min[0], scene.bounds.min[1], scene.bounds.min[2]};
  const double bmax[3] = {scene.bounds.max[0], scene.bounds.max[1], scene.bounds.max[2]};
  check(gavis_active_mapping(detail::holder().get(), ds->h, bmin, bmax, rects.data(),
                             (int32_t)rects.size(), occluders.sample_density, init_c.data(),
                             (int32_t)init_c.size(), &g, &mc, chosen.data(), idx.data(),
                             score.data(), all.data(), cov.data(), ment.data()));
  MappingLog log;
  for (int s = 0; s < steps; ++s) {
    log.chosen_views.views.push_back(detail::cam_from_c(chosen[s]));
    MappingStep st;
    st.scores.assign(all.begin() + (size_t)s * nc, all.begin() + (size_t)(s + 1) * nc);
    st.chosen_index = idx[s];
    st.score = score[s];
    st.vis_coverage = cov[s];
    st.mean_entropy = ment[s];
    log.steps.push_back(std::move(st));
  }
  return log;
}

// ---- device-resident handles ------------------------------------------------
// The reference-signature functions above take host values and upload the scene
// (and field) per call. A planner loop (planner.hpp:297-301) that scores many
// candidate sets against one scene keeps them resident instead: upload once,
// then call the overloads below with the handles (no per-call H2D of the scene
// or field).
class ResidentScene {
 public:
  explicit ResidentScene(const Scene& s, const UncertaintyConfig* uc = nullptr)
      : dev_(detail::upload(s)), n_(s.particles.size()), virt_(detail::virtual_mask(s)) {
    if (uc) detail::attach_variances(*uc, dev_->h, n_);
  }
  // attach UncertaintyConfig::coeff_variances (kShPropagation) after the fact
  void set_variances(const UncertaintyConfig& uc) { detail::attach_variances(uc, dev_->h, n_); }
  gavis_scene* handle() const { return dev_->h; }
  std::size_t size() const { return n_; }
  const std::vector<uint8_t>& virtual_mask() const { return virt_; }

 private:
  std::unique_ptr<detail::DeviceScene> dev_;
  std::size_t n_;
  std::vector<uint8_t> virt_;
};

class ResidentField {
 public:
  ResidentField(const ResidentScene& s, gavis_field* h, int degree, const VmfParams& vmf)
      : scene_(&s), degree_(degree), vmf_(vmf) {
    dev_.h = h;
  }
  // a host field (e.g. load_field) made resident
  ResidentField(const ResidentScene& s, const VisibilityField& f)
      : scene_(&s), degree_(f.degree), vmf_(f.vmf) {
    if (f.num_particles != s.size()) throw ParameterError("field was built for a different scene");
    check(gavis_vf_upload(detail::holder().get(), s.handle(), f.vmf.kappa, f.degree, f.num_views,
                          f.gamma.empty() ? nullptr : f.gamma.data(), &dev_.h));
  }
  ResidentField(const ResidentField&) = delete;
  ResidentField& operator=(const ResidentField&) = delete;
  ResidentField(ResidentField&& o) noexcept : scene_(o.scene_), degree_(o.degree_), vmf_(o.vmf_) {
    dev_.h = o.dev_.h;
    o.dev_.h = nullptr;
  }
  gavis_field* handle() const { return dev_.h; }
  const ResidentScene& scene() const { return *scene_; }
  int num_views() const {
    int32_t nv = 0;
    check(gavis_vf_download(dev_.h, nullptr, &nv, nullptr));
    return nv;
  }
  // appends views (vfield.hpp:38-63 per view, num_views += views)
  void accumulate(const Trajectory& views, const RasterConfig& rc = {}) {
    std::vector<gavis_camera> cams;
    for (const auto& v : views.views) cams.push_back(detail::cam_c(v));
    const gavis_raster_config r = detail::rc_c(rc);
    check(gavis_vf_accumulate_views(detail::holder().get(), dev_.h, scene_->handle(), cams.data(),
                                    (int32_t)cams.size(), &r));
  }
  VisibilityField download() const {
    VisibilityField out;
    out.degree = degree_;
    out.vmf = vmf_;
    out.num_particles = scene_->size();
    out.gamma.resize(out.num_particles * out.basis_size());
    int32_t nv = 0;
    check(gavis_vf_download(dev_.h, out.gamma.empty() ? nullptr : out.gamma.data(), &nv, nullptr));
    out.num_views = nv;
    out.virtual_mask = scene_->virtual_mask();
    return out;
  }

 private:
  const ResidentScene* scene_;
  int degree_;
  VmfParams vmf_;
  detail::DeviceField dev_;
};

// vfield.hpp:68-92 on a resident scene; the field stays on the device.
inline ResidentField construct_field(const ResidentScene& scene, const Trajectory& trajectory,
                                     const VmfParams& vmf, int degree, const RasterConfig& rc = {}) {
  std::vector<gavis_camera> cams;
  for (const auto& v : trajectory.views) cams.push_back(detail::cam_c(v));
  const gavis_raster_config r = detail::rc_c(rc);
  gavis_field* f = nullptr;
  check(gavis_vf_construct(detail::holder().get(), scene.handle(), cams.data(), (int32_t)cams.size(),
                           vmf.kappa, degree, &r, &f));
  return ResidentField(scene, f, degree, vmf);
}

// uncertainty.hpp:242-260 on resident handles (entropy map + optional entropy depth)
inline EntropyMap render_entropy(const ResidentScene& scene, const ResidentField& field,
                                 const CameraView& cam, const RasterConfig& rc,
                                 const UncertaintyConfig& uc, std::vector<double>* depth_out = nullptr) {
  const gavis_camera c = detail::cam_c(cam);
  const gavis_raster_config r = detail::rc_c(rc);
  const gavis_uncertainty_config u = detail::uc_c(uc);
  EntropyMap m;
  m.width = cam.width;
  m.height = cam.height;
  const std::size_t P = (std::size_t)cam.width * cam.height;
  m.entropy.resize(P);
  m.invisible_mass.resize(P);
  if (depth_out) depth_out->resize(P);
  gavis_render_outputs o{};
  o.entropy = m.entropy.data();
  o.invisible_mass = m.invisible_mass.data();
  o.entropy_depth = depth_out ? depth_out->data() : nullptr;
  check(gavis_ua_render(detail::holder().get(), scene.handle(), field.handle(), nullptr, &c, 1, &r, &u, &o));
  return m;
}

// planner.hpp:117-137 on resident handles
inline NbvResult select_nbv(const ResidentScene& scene, const ResidentField& field,
                            const std::vector<CameraView>& candidates, const RasterConfig& rc,
                            const UncertaintyConfig& uc) {
  if (candidates.empty()) throw ParameterError("select_nbv: candidate list must be nonempty");
  std::vector<gavis_camera> cams;
  for (const auto& v : candidates) cams.push_back(detail::cam_c(v));
  const gavis_raster_config r = detail::rc_c(rc);
  const gavis_uncertainty_config u = detail::uc_c(uc);
  NbvResult res;
  res.scores.resize(candidates.size());
  int32_t best = -1;
  check(gavis_select_nbv(detail::holder().get(), scene.handle(), field.handle(), cams.data(),
                         (int32_t)cams.size(), &r, &u, 0, res.scores.data(), &best));
  res.best_index = best;
  return res;
}

// ---- multi-GPU (one process per GPU) ------------------------------
// Rank 0 makes the id (Communicator::unique_id), the host ships the bytes to the
// other ranks (MPI, a file, a socket), every rank builds its Communicator on its
// own device (set_default_device first).
class Communicator {
 public:
  using Id = std::array<uint8_t, GAVIS_COMM_ID_BYTES>;
  static Id unique_id() {
    Id id{};
    check(gavis_comm_unique_id(id.data()));
    return id;
  }
  Communicator(const Id& id, int nranks, int rank) : nranks_(nranks), rank_(rank) {
    check(gavis_comm_create(detail::holder().get(), id.data(), nranks, rank, &h_));
  }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  ~Communicator() {
    if (h_) gavis_comm_destroy(h_);
  }
  gavis_comm* handle() const { return h_; }
  int nranks() const { return nranks_; }
  int rank() const { return rank_; }

 private:
  gavis_comm* h_ = nullptr;
  int nranks_, rank_;
};

// construct_field with the trajectory split in static blocks over the ranks
// (the reference's parallel_for over views, vfield.hpp:85-90) and the partial
// fields all-reduced over NCCL. Collective.
inline ResidentField construct_field_sharded(const Communicator& comm, const ResidentScene& scene,
                                             const Trajectory& trajectory, const VmfParams& vmf,
                                             int degree, const RasterConfig& rc = {}) {
  std::vector<gavis_camera> cams;
  for (const auto& v : trajectory.views) cams.push_back(detail::cam_c(v));
  const gavis_raster_config r = detail::rc_c(rc);
  gavis_field* f = nullptr;
  check(gavis_vf_construct_sharded(comm.handle(), scene.handle(), cams.data(), (int32_t)cams.size(),
                                   vmf.kappa, degree, &r, &f));
  return ResidentField(scene, f, degree, vmf);
}

// select_nbv with the candidates split in static blocks over the ranks
// (planner.hpp:125-131); every rank returns all scores and the same index. Collective.
inline NbvResult select_nbv_sharded(const Communicator& comm, const ResidentScene& scene,
                                    const ResidentField& field, const std::vector<CameraView>& candidates,
                                    const RasterConfig& rc, const UncertaintyConfig& uc) {
  if (candidates.empty()) throw ParameterError("select_nbv: candidate list must be nonempty");
  std::vector<gavis_camera> cams;
  for (const auto& v : candidates) cams.push_back(detail::cam_c(v));
  const gavis_raster_config r = detail::rc_c(rc);
  const gavis_uncertainty_config u = detail::uc_c(uc);
  NbvResult res;
  res.scores.resize(candidates.size());
  int32_t best = -1;
  check(gavis_select_nbv_sharded(comm.handle(), scene.handle(), field.handle(), cams.data(),
                                 (int32_t)cams.size(), &r, &u, 0, res.scores.data(), &best));
  res.best_index = best;
  return res;
}

}  // namespace gavis_b200
