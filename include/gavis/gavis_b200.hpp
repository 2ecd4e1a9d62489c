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

// uncertainty.hpp:24-52 (constant provider, no correlation hook)
struct UncertaintyConfig {
  double beta = 0.5;
  double prior_opacity = 0.15;
  Mat3 prior_cov;
  double color_sigma = 0.1;
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
  g.correlation_lambda = 1.0;
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
                                 std::vector<double>* depth_out = nullptr) {
  if (field.num_particles != scene.particles.size())
    throw ParameterError("render_entropy: field was built for a different scene");
  auto ds = detail::upload(scene);
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
  return m;
}

// uncertainty.hpp:264-272 (correlation none)
inline double image_entropy(const EntropyMap& map, const std::vector<double>& depth,
                            const UncertaintyConfig& /*uc*/) {
  if (depth.size() != map.entropy.size())
    throw ParameterError("image_entropy: depth map shape differs from the entropy map");
  double sum = 0.0;
  for (double h : map.entropy) sum += h;
  return sum;
}

// planner.hpp:117-137
inline NbvResult select_nbv(const Scene& scene_aug, const VisibilityField& field,
                            const std::vector<CameraView>& candidates, const RasterConfig& rc,
                            const UncertaintyConfig& uc, int /*threads*/ = 1) {
  if (candidates.empty()) throw ParameterError("select_nbv: candidate list must be nonempty");
  auto ds = detail::upload(scene_aug);
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

}  // namespace gavis_b200
