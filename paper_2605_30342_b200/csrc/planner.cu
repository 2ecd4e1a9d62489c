// planner.cu -- the callers of the hot path in the reference planner
// (R/include/gavis/planner.hpp), host C++ around the device entry points:
//   * sample_candidates (planner.hpp:56-107): rejection-sampled candidate poses;
//   * vis_coverage (planner.hpp:155-184): occluder-surface coverage metric;
//   * run_active_mapping (planner.hpp:284-316): density control -> field
//     rebuild -> candidate sampling -> select_nbv -> append, per step.
// Geometry follows the reference's double expressions in order; the Eigen
// fixed-size kernels it relies on are restated explicitly (3x3 determinant and
// cofactor inverse, quaternion normalisation, toRotationMatrix).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "gavis_b200.h"

namespace gavis {
void set_last_error(const std::string& msg);  // gavis_abi.cu
}

namespace {

constexpr double kPi = 3.14159265358979323846;  // common.hpp:20

struct PlanErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StatusErr {
  gavis_status s;
};

void need(bool c, const std::string& m) {
  if (!c) throw PlanErr(m);
}
void ok(gavis_status s) {
  if (s != GAVIS_OK) throw StatusErr{s};  // callee already set gavis_last_error
}

template <class F>
gavis_status plan_guard(F&& f) {
  try {
    f();
    return GAVIS_OK;
  } catch (const StatusErr& e) {
    return e.s;
  } catch (const PlanErr& e) {
    gavis::set_last_error(e.what());
    return GAVIS_ERR_PARAMETER;
  } catch (const std::bad_alloc&) {
    gavis::set_last_error("host allocation failed");
    return GAVIS_ERR_DEVICE;
  }
}

struct V3 {
  double x, y, z;
};
V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
double norm(V3 a) { return std::sqrt(dot(a, a)); }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
V3 normalized(V3 a) {
  const double n = norm(a);
  return {a.x / n, a.y / n, a.z / n};
}
V3 load3(const double* p) { return {p[0], p[1], p[2]}; }

// rng.hpp:18-89
uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ mix64(stream + 0x632be59bd9b4e019ull));
}
struct Rng {
  uint64_t s;
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return (double)(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
  // Shoemake (rng.hpp:77-85): (w, x, y, z)
  void rotation(double q[4]) {
    const double u1 = unit(), u2 = unit(), u3 = unit();
    const double a = std::sqrt(1.0 - u1), b = std::sqrt(u1);
    q[0] = a * std::sin(2.0 * kPi * u2);
    q[1] = a * std::cos(2.0 * kPi * u2);
    q[2] = b * std::sin(2.0 * kPi * u3);
    q[3] = b * std::cos(2.0 * kPi * u3);
  }
};

void set_rotation_cols(gavis_camera& v, V3 c0, V3 c1, V3 c2) {
  const V3 cols[3] = {c0, c1, c2};
  for (int c = 0; c < 3; ++c) {
    v.rotation[0 * 3 + c] = cols[c].x;
    v.rotation[1 * 3 + c] = cols[c].y;
    v.rotation[2 * 3 + c] = cols[c].z;
  }
}

// make_lookat (model.hpp:107-128), default up (0, 0, 1).
gavis_camera make_lookat(V3 position, V3 target) {
  V3 forward = target - position;
  need(norm(forward) > 1e-12, "lookat target coincides with position");
  forward = normalized(forward);
  V3 right = cross(forward, V3{0.0, 0.0, 1.0});
  if (norm(right) < 1e-9) right = cross(forward, V3{1.0, 0.0, 0.0});
  right = normalized(right);
  const V3 down = cross(forward, right);
  gavis_camera v{};
  set_rotation_cols(v, right, down, forward);
  v.position[0] = position.x;
  v.position[1] = position.y;
  v.position[2] = position.z;
  return v;
}

// q.normalized().toRotationMatrix(): Eigen stores (x, y, z, w); its SSE2
// squaredNorm of the 4 coefficients sums (x^2 + z^2) + (y^2 + w^2).
void quat_to_rotation(const double qw[4], double R[9]) {
  const double w0 = qw[0], x0 = qw[1], y0 = qw[2], z0 = qw[3];
  const double n = std::sqrt((x0 * x0 + z0 * z0) + (y0 * y0 + w0 * w0));
  const double w = w0 / n, x = x0 / n, y = y0 / n, z = z0 / n;
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0] = 1 - (tyy + tzz);
  R[1] = txy - twz;
  R[2] = txz + twy;
  R[3] = txy + twz;
  R[4] = 1 - (txx + tzz);
  R[5] = tyz - twx;
  R[6] = txz - twy;
  R[7] = tyz + twx;
  R[8] = 1 - (txx + tyy);
}

struct Rect {
  V3 corner, eu, ev;
  bool opaque;
};
Rect load_rect(const gavis_occluder_rect& r) {
  return {load3(r.corner), load3(r.edge_u), load3(r.edge_v), r.opaque != 0};
}
V3 point_at(const Rect& r, double u, double v) { return (r.corner + u * r.eu) + v * r.ev; }

// rect_distance (planner.hpp:45-52)
double rect_distance(const Rect& r, V3 p) {
  const V3 w = p - r.corner;
  const double uu = dot(r.eu, r.eu), vv = dot(r.ev, r.ev);
  const double u = uu > 0.0 ? std::clamp(dot(w, r.eu) / uu, 0.0, 1.0) : 0.0;
  const double v = vv > 0.0 ? std::clamp(dot(w, r.ev) / vv, 0.0, 1.0) : 0.0;
  return norm(point_at(r, u, v) - p);
}

// intersect_rect (model.hpp:157-175): m = [eu | ev | -dir], Eigen's 3x3
// determinant and cofactor inverse, sol = m^-1 (origin - corner).
bool intersect_rect(const Rect& r, V3 origin, V3 dir, double* t_out) {
  const double m[3][3] = {{r.eu.x, r.ev.x, -dir.x}, {r.eu.y, r.ev.y, -dir.y}, {r.eu.z, r.ev.z, -dir.z}};
  auto det3 = [&](int a, int b, int c) { return m[0][a] * (m[1][b] * m[2][c] - m[1][c] * m[2][b]); };
  const double det = det3(0, 1, 2) - det3(1, 0, 2) + det3(2, 0, 1);
  if (std::abs(det) < 1e-14) return false;
  auto cof = [&](int i, int j) {
    const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
    return m[i1][j1] * m[i2][j2] - m[i1][j2] * m[i2][j1];
  };
  const double c00 = cof(0, 0), c10 = cof(1, 0), c20 = cof(2, 0);
  const double d = (c00 * m[0][0] + c10 * m[1][0]) + c20 * m[2][0];
  const double invdet = 1.0 / d;
  double inv[3][3];
  inv[0][0] = c00 * invdet;
  inv[0][1] = c10 * invdet;
  inv[0][2] = c20 * invdet;
  inv[1][0] = cof(0, 1) * invdet;
  inv[1][1] = cof(1, 1) * invdet;
  inv[1][2] = cof(2, 1) * invdet;
  inv[2][0] = cof(0, 2) * invdet;
  inv[2][1] = cof(1, 2) * invdet;
  inv[2][2] = cof(2, 2) * invdet;
  const V3 w = origin - r.corner;
  const double u = inv[0][0] * w.x + inv[0][1] * w.y + inv[0][2] * w.z;
  const double v = inv[1][0] * w.x + inv[1][1] * w.y + inv[1][2] * w.z;
  const double t = inv[2][0] * w.x + inv[2][1] * w.y + inv[2][2] * w.z;
  if (u < 0.0 || u > 1.0 || v < 0.0 || v > 1.0) return false;
  *t_out = t;
  return true;
}

// CameraView::project (model.hpp:90-97)
bool project(const gavis_camera& c, V3 p) {
  const V3 d = p - load3(c.position);
  const double* R = c.rotation;  // camera = R^T d
  const double cx_ = R[0] * d.x + R[3] * d.y + R[6] * d.z;
  const double cy_ = R[1] * d.x + R[4] * d.y + R[7] * d.z;
  const double cz_ = R[2] * d.x + R[5] * d.y + R[8] * d.z;
  if (cz_ < c.near_plane) return false;
  const double fx = 0.5 * c.width / std::tan(0.5 * c.fov_h);
  const double fy = 0.5 * c.height / std::tan(0.5 * c.fov_v);
  const double px = 0.5 * c.width + fx * cx_ / cz_;
  const double py = 0.5 * c.height + fy * cy_ / cz_;
  return px >= 0.0 && px <= c.width && py >= 0.0 && py <= c.height;
}

// point_visible_from_view (planner.hpp:141-153)
bool point_visible(V3 point, const gavis_camera& view, const std::vector<Rect>& rects, int exclude) {
  if (!project(view, point)) return false;
  const V3 pos = load3(view.position);
  const V3 seg = point - pos;
  for (size_t j = 0; j < rects.size(); ++j) {
    if (!rects[j].opaque || (int)j == exclude) continue;
    double t;
    if (intersect_rect(rects[j], pos, seg, &t) && t > 1e-9 && t < 1.0 - 1e-9) return false;
  }
  return true;
}

double coverage(const std::vector<Rect>& rects, double density, const gavis_camera* views, int n_views) {
  double total = 0.0, visible = 0.0;
  for (size_t r = 0; r < rects.size(); ++r) {
    const Rect& rc = rects[r];
    const double area = norm(cross(rc.eu, rc.ev));
    need(area > 0.0, "vis_coverage: occluder rectangle with zero area");
    total += area;
    if (n_views == 0) continue;
    const double per_side = std::sqrt(density);
    const int nu = std::max(1, (int)std::lround(norm(rc.eu) * per_side));
    const int nv = std::max(1, (int)std::lround(norm(rc.ev) * per_side));
    long long seen = 0;
    for (int i = 0; i < nu; ++i)
      for (int j = 0; j < nv; ++j) {
        const V3 p = point_at(rc, (i + 0.5) / nu, (j + 0.5) / nv);
        for (int k = 0; k < n_views; ++k)
          if (point_visible(p, views[k], rects, (int)r)) {
            ++seen;
            break;
          }
      }
    visible += area * (double)seen / ((double)nu * nv);
  }
  return total > 0.0 ? visible / total : 0.0;
}

void validate_planner(const gavis_planner_config* pc) {
  need(pc != nullptr, "null planner config");
  need(pc->num_candidates >= 1, "num_candidates must be at least 1");
  need(pc->steps >= 0, "steps must be non-negative");
  need(pc->mode == 0 || pc->mode == 1, "pose mode must be 0 (SE3) or 1 (SE2)");
}

void sample(const double* bmin, const double* bmax, const std::vector<Rect>& rects,
            const gavis_planner_config* pc, uint64_t step_seed, gavis_camera* out) {
  validate_planner(pc);
  const V3 lo = load3(bmin), hi = load3(bmax);
  const V3 ext = hi - lo;
  need(ext.x * ext.y * ext.z > 0.0, "sample_candidates: bounds volume must be positive");
  Rng g{derive_seed(step_seed, 0xca4d1d)};
  const long long budget = 100LL * pc->num_candidates;
  long long attempts = 0;
  int n = 0;
  while (n < pc->num_candidates) {
    if (attempts++ >= budget) throw PlanErr("candidate sampling budget exhausted; scene too cluttered");
    V3 p;
    // planner.hpp:70-72 draws the coordinates as the arguments of one Vec3
    // constructor call (evaluation order unspecified by C++); the reference's GCC
    // build evaluates them right to left -- z, y, x -- and so do we, so the
    // candidates equal the reference binary's bit for bit (tests/test_planner.py)
    p.z = g.uniform(lo.z, hi.z);
    p.y = g.uniform(lo.y, hi.y);
    p.x = g.uniform(lo.x, hi.x);
    const double yaw = g.uniform(0.0, 2.0 * kPi);  // drawn in both modes
    double q[4];
    g.rotation(q);
    if (pc->mode == 1) p.z = pc->se2_height;
    bool collides = false;
    for (const Rect& r : rects) {
      if (!r.opaque) continue;
      if (rect_distance(r, p) < pc->clearance) {
        collides = true;
        break;
      }
    }
    if (collides) continue;
    gavis_camera view{};
    if (pc->mode == 1) {
      const V3 forward{std::cos(yaw), std::sin(yaw), 0.0};
      view = make_lookat(p, p + forward);
    } else if (pc->look_inward) {
      V3 target = 0.5 * (lo + hi);
      if (norm(target - p) < 1e-9) target = target + V3{1e-3, 0.0, 0.0};
      view = make_lookat(p, target);
    } else {
      quat_to_rotation(q, view.rotation);
    }
    view.position[0] = p.x;
    view.position[1] = p.y;
    view.position[2] = p.z;
    view.width = pc->cam_width;
    view.height = pc->cam_height;
    view.fov_h = pc->fov_h;
    view.fov_v = pc->fov_v;
    view.near_plane = pc->cam_near;
    out[n++] = view;
  }
}

std::vector<Rect> load_rects(const gavis_occluder_rect* rects, int32_t n) {
  need(n >= 0 && (rects != nullptr || n == 0), "occluder rectangles must not be null");
  std::vector<Rect> out;
  out.reserve(n);
  for (int i = 0; i < n; ++i) out.push_back(load_rect(rects[i]));
  return out;
}

}  // namespace

extern "C" {

gavis_status gavis_sample_candidates(const double* bounds_min, const double* bounds_max,
                                     const gavis_occluder_rect* rects, int32_t n_rects,
                                     const gavis_planner_config* pc, uint64_t step_seed,
                                     gavis_camera* out) {
  return plan_guard([&] {
    need(bounds_min && bounds_max && out, "null argument");
    sample(bounds_min, bounds_max, load_rects(rects, n_rects), pc, step_seed, out);
  });
}

gavis_status gavis_vis_coverage(const gavis_occluder_rect* rects, int32_t n_rects,
                                double sample_density, const gavis_camera* views,
                                int32_t n_views, double* cov) {
  return plan_guard([&] {
    need(cov != nullptr, "null argument");
    need(n_views >= 0 && (views != nullptr || n_views == 0), "views must not be null");
    *cov = coverage(load_rects(rects, n_rects), sample_density, views, n_views);
  });
}

gavis_status gavis_active_mapping(gavis_ctx* ctx, const gavis_scene* scene,
                                  const double* bounds_min, const double* bounds_max,
                                  const gavis_occluder_rect* rects, int32_t n_rects,
                                  double sample_density, const gavis_camera* init_views,
                                  int32_t n_init, const gavis_planner_config* pc,
                                  const gavis_mapping_config* mc, gavis_camera* chosen_views,
                                  int32_t* chosen_index, double* chosen_score,
                                  double* all_scores, double* vis_cov, double* mean_entropy) {
  return plan_guard([&] {
    need(ctx && scene && bounds_min && bounds_max && mc, "null argument");
    validate_planner(pc);
    need(n_init >= 1 && init_views != nullptr,
         "run_active_mapping: initial trajectory must be nonempty");
    const std::vector<Rect> occ = load_rects(rects, n_rects);
    std::vector<gavis_camera> traj(init_views, init_views + n_init);
    std::vector<gavis_camera> cands(pc->num_candidates);
    std::vector<double> scores(pc->num_candidates);
    for (int step = 0; step < pc->steps; ++step) {
      gavis_scene* aug = nullptr;
      gavis_field* field = nullptr;
      try {
        const gavis_scene* sc = scene;
        if (mc->density_enabled) {
          gavis_density_config dc = mc->density;
          dc.seed = derive_seed(mc->density.seed, (uint64_t)step);
          int64_t kept = 0;
          ok(gavis_density_control(ctx, scene, bounds_min, bounds_max, traj.data(), (int32_t)traj.size(),
                                   &dc, &mc->raster, &aug, &kept, nullptr, 0));
          sc = aug;
        }
        ok(gavis_vf_construct(ctx, sc, traj.data(), (int32_t)traj.size(), mc->kappa, mc->field_degree,
                              &mc->raster, &field));
        sample(bounds_min, bounds_max, occ, pc, derive_seed(pc->seed, (uint64_t)step), cands.data());
        int32_t best = -1;
        ok(gavis_select_nbv(ctx, sc, field, cands.data(), pc->num_candidates, &mc->raster,
                            &mc->uncertainty, 0, scores.data(), &best));
        const gavis_camera& ch = cands[best];
        traj.push_back(ch);
        if (chosen_views) chosen_views[step] = ch;
        if (chosen_index) chosen_index[step] = best;
        if (chosen_score) chosen_score[step] = scores[best];
        if (all_scores)
          std::memcpy(all_scores + (size_t)step * pc->num_candidates, scores.data(),
                      sizeof(double) * pc->num_candidates);
        if (vis_cov) vis_cov[step] = coverage(occ, sample_density, traj.data(), (int)traj.size());
        if (mean_entropy) mean_entropy[step] = scores[best] / ((double)ch.width * ch.height);
      } catch (...) {
        if (field) gavis_vf_destroy(field);
        if (aug) gavis_scene_destroy(aug);
        throw;
      }
      gavis_vf_destroy(field);
      if (aug) gavis_scene_destroy(aug);
    }
  });
}

}  // extern "C"
