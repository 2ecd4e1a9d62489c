// dropin_check.cpp -- test infrastructure (built only where /root/reference is
// present: `make -C oracle ref`, output oracle/_ref/dropin_check; run on a GPU
// box by tests/test_cpp_frontend.py::test_dropin_source_compatible_with_reference).
//
// One templated caller, written the way planner.hpp:297-301 and the CLI call the
// reference (Scene of GaussianParticle, Trajectory, construct_field,
// select_nbv), instantiated twice: with namespace gavis (the reference's own
// headers, CPU) and with namespace gavis_b200 (include/gavis/gavis_b200.hpp,
// the drop-in over libgavis_b200.so). Switching a reference caller over is the
// namespace (plus the quaternion type's construction); both runs must pick the
// same view with the same scores.
#include <gavis/planner.hpp>
#include <gavis/vfield.hpp>

#include <gavis/gavis_b200.hpp>

#include <cmath>
#include <cstdio>
#include <vector>

namespace {

uint64_t next(uint64_t& s) {
  s += 0x9e3779b97f4a7c15ull;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// scene values are drawn fp32-representable: the drop-in stores the scene as fp32
// SoA on the device (the C ABI's layout), the reference keeps doubles
double unit(uint64_t& s) { return (double)(float)((double)(next(s) >> 11) * 0x1.0p-53); }
double f32(double x) { return (double)(float)x; }

template <class Q>
Q quat(double w, double x, double y, double z);
template <>
gavis::Quat quat<gavis::Quat>(double w, double x, double y, double z) { return gavis::Quat(w, x, y, z); }
template <>
gavis_b200::Quat quat<gavis_b200::Quat>(double w, double x, double y, double z) {
  gavis_b200::Quat q;
  q.w = w, q.x = x, q.y = y, q.z = z;
  return q;
}

// The same caller code for both APIs.
template <class Scene, class Particle, class Quat, class Vec3, class Traj, class Vmf, class Raster, class Unc,
          class MakeLookat, class Construct, class Select>
std::vector<double> plan(int& best, MakeLookat make_lookat, Construct construct_field, Select select_nbv) {
  Scene scene;
  scene.color_degree = 1;
  uint64_t s = 12345;
  for (int i = 0; i < 3000; ++i) {
    Particle p;
    const double px = f32(-1.5 + 3.0 * unit(s)), py = f32(-1.5 + 3.0 * unit(s)), pz = f32(2.0 + 3.0 * unit(s));
    p.position = Vec3(px, py, pz);
    const double a = unit(s), b = unit(s), c = unit(s);
    const double r1 = std::sqrt(1 - a), r2 = std::sqrt(a);
    p.rotation = quat<Quat>(f32(r1 * std::sin(6.283185307179586 * b)), f32(r1 * std::cos(6.283185307179586 * b)),
                            f32(r2 * std::sin(6.283185307179586 * c)), f32(r2 * std::cos(6.283185307179586 * c)));
    const double sc = f32(std::exp(-3.5 + 0.5 * unit(s))), sy = f32(sc * (0.5 + unit(s)));
    p.scale = Vec3(sc, sy, sc);
    p.opacity = f32(0.2 + 0.7 * unit(s));
    for (int ch = 0; ch < 3; ++ch) {
      p.color_sh[ch].assign(4, 0.0);
      for (int k = 0; k < 4; ++k) p.color_sh[ch][k] = f32(0.3 * (unit(s) - 0.5) + (k == 0 ? 1.7 : 0.0));
    }
    scene.particles.push_back(p);
  }
  Traj traj;
  for (int v = 0; v < 6; ++v)
    traj.views.push_back(make_lookat(Vec3(-0.6 + 0.24 * v, 0.2, -0.5), Vec3(0, 0, 3.5), Vec3(0, -1, 0), 96, 80,
                                     1.2, 1.0));
  std::vector<typename std::decay<decltype(traj.views[0])>::type> cands;
  for (int v = 0; v < 8; ++v)
    cands.push_back(make_lookat(Vec3(0.9 * std::cos(0.7 * v), 0.9 * std::sin(0.7 * v), 0.0), Vec3(0, 0, 3.5),
                                Vec3(0, -1, 0), 96, 80, 1.2, 1.0));
  const Raster rc;
  const Unc uc;
  const auto field = construct_field(scene, traj, Vmf(1.0), 2, rc, 4);
  const auto nbv = select_nbv(scene, field, cands, rc, uc, 4);
  best = nbv.best_index;
  return nbv.scores;
}

}  // namespace

int main() {
  int best_r = -1, best_b = -1;
  const std::vector<double> sr =
      plan<gavis::Scene, gavis::GaussianParticle, gavis::Quat, gavis::Vec3, gavis::Trajectory, gavis::VmfParams,
           gavis::RasterConfig, gavis::UncertaintyConfig>(
          best_r, [](auto... a) { return gavis::make_lookat(a...); },
          [](auto&&... a) { return gavis::construct_field(a...); },
          [](auto&&... a) { return gavis::select_nbv(a...); });
  const std::vector<double> sb =
      plan<gavis_b200::Scene, gavis_b200::GaussianParticle, gavis_b200::Quat, gavis_b200::Vec3,
           gavis_b200::Trajectory, gavis_b200::VmfParams, gavis_b200::RasterConfig, gavis_b200::UncertaintyConfig>(
          best_b, [](auto... a) { return gavis_b200::make_lookat(a...); },
          [](auto&&... a) { return gavis_b200::construct_field(a...); },
          [](auto&&... a) { return gavis_b200::select_nbv(a...); });
  double rel = 0.0;
  for (size_t i = 0; i < sr.size() && i < sb.size(); ++i)
    rel = std::max(rel, std::fabs(sr[i] - sb[i]) / std::max(1e-300, std::fabs(sr[i])));
  std::printf("reference_best %d b200_best %d candidates %zu %zu max_score_rel %.3e\n", best_r, best_b, sr.size(),
              sb.size(), rel);
  return (best_r == best_b && sr.size() == sb.size() && rel <= 1e-9) ? 0 : 1;
}
