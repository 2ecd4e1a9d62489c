// Reference-shaped caller of the drop-in C++ API exercising the non-default
// UncertaintyConfig paths (uncertainty.hpp:24-52): the sh_propagation variance
// provider with per-particle coefficient variances (:62-83, :149-163) and the
// correlation hook of image_entropy (:264-278), through
//   * the reference signatures (host values, uploaded per call),
//   * the device-resident handles (planner.hpp:297-301 without re-uploads),
//   * the sharded entry points on a one-rank communicator (NCCL).
// The scene is built from closed-form formulas that tests/test_cpp_frontend.py
// repeats in Python to check the printed scores against the CPU oracle.
#include <cstdio>
#include <cstring>

#include "gavis/gavis_b200.hpp"

using namespace gavis_b200;

static Scene make_scene() {
  Scene scene;
  scene.color_degree = 1;
  int k = 0;
  auto colors = [&](GaussianParticle& g) {
    for (int c = 0; c < 3; ++c)
      g.color_sh[c] = {(0.3 + 0.1 * c) / kY00, 0.1 * ((k + c) % 3 - 1), 0.05 * (k % 4), -0.02 * c};
    ++k;
  };
  for (int i = 0; i < 7; ++i)
    for (int j = 0; j < 7; ++j) {
      GaussianParticle g;
      g.position = Vec3(1.0, 0.2 + 0.1 * i, 0.2 + 0.1 * j);
      g.scale = Vec3(0.05, 0.06, 0.04);
      g.opacity = 0.85;
      colors(g);
      scene.particles.push_back(g);
    }
  for (int m = 0; m < 30; ++m) {
    GaussianParticle g;
    g.position = Vec3(1.2 + 0.05 * (m % 5), 0.2 + 0.07 * (m % 9), 0.25 + 0.06 * (m % 8));
    g.scale = Vec3(0.03, 0.03, 0.03);
    g.opacity = 0.5 + 0.01 * m;
    colors(g);
    scene.particles.push_back(g);
  }
  return scene;
}

static std::vector<std::array<std::vector<double>, 3>> make_variances(std::size_t n) {
  std::vector<std::array<std::vector<double>, 3>> v(n);
  for (std::size_t i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c)
      for (int m = 0; m < 4; ++m) v[i][c].push_back(0.001 * (1 + (int)((i + c + m) % 5)));
  return v;
}

static void print(const char* tag, const NbvResult& r) {
  std::printf("%s best %d", tag, r.best_index);
  for (double s : r.scores) std::printf(" %.17g", s);
  std::printf("\n");
}

int main(int argc, char** argv) {
  if (argc > 1) set_exact_precision(std::strcmp(argv[1], "exact") == 0);  // "exact" | "certified"
  try {
    const Scene scene = make_scene();
    const auto variances = make_variances(scene.particles.size());
    const CameraView front = make_lookat(Vec3(0.3, 0.5, 0.5), Vec3(1, 0.5, 0.5), Vec3(0, 0, 1), 64, 64);
    const std::vector<CameraView> cands = {
        front, make_lookat(Vec3(1.9, 0.5, 0.5), Vec3(1, 0.5, 0.5), Vec3(0, 0, 1), 64, 64),
        make_lookat(Vec3(1.1, -0.6, 0.5), Vec3(1.1, 0.5, 0.5), Vec3(0, 0, 1), 64, 64),
        make_lookat(Vec3(0.6, 0.1, 0.9), Vec3(1.1, 0.5, 0.5), Vec3(0, 0, 1), 64, 64)};
    Trajectory traj;
    traj.views = {front};
    const VisibilityField field = construct_field(scene, traj, VmfParams(1.0), 2);

    UncertaintyConfig sh;
    sh.variance_provider = VarianceProvider::kShPropagation;
    sh.coeff_variances = &variances;
    UncertaintyConfig hook;
    hook.correlation = CorrelationMode::kHook;
    hook.correlation_lambda = 0.7;
    UncertaintyConfig both = sh;
    both.correlation = CorrelationMode::kHook;
    both.correlation_lambda = 0.7;

    // 1. reference signatures
    print("sh", select_nbv(scene, field, cands, RasterConfig{}, sh));
    print("hook", select_nbv(scene, field, cands, RasterConfig{}, hook));
    print("both", select_nbv(scene, field, cands, RasterConfig{}, both));
    // image_entropy with the hook from the maps (host fold) vs the device score
    std::vector<double> depth;
    const EntropyMap m = render_entropy(scene, field, cands[1], RasterConfig{}, both, 1, &depth);
    std::printf("image_entropy_hook %.17g\n", image_entropy(m, depth, both));

    // 2. resident handles: one upload, several scorings
    ResidentScene rs(scene, &sh);
    ResidentField rf = construct_field(rs, traj, VmfParams(1.0), 2);
    print("resident_both", select_nbv(rs, rf, cands, RasterConfig{}, both));

    // 3. sharded entry points on one rank
    Communicator comm(Communicator::unique_id(), 1, 0);
    ResidentField sf = construct_field_sharded(comm, rs, traj, VmfParams(1.0), 2);
    print("sharded_both", select_nbv_sharded(comm, rs, sf, cands, RasterConfig{}, both));
    const VisibilityField back = sf.download();
    double dmax = 0.0;
    for (std::size_t i = 0; i < back.gamma.size(); ++i)
      dmax = std::max(dmax, std::fabs(back.gamma[i] - field.gamma[i]));
    std::printf("sharded_field_max_abs %.3g num_views %d\n", dmax, back.num_views);
    return 0;
  } catch (const DeviceError& e) {
    std::printf("device error: %s\n", e.what());
    return 5;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 2;
  }
}
