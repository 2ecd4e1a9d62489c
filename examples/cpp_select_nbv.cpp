// Reference-style caller of the drop-in C++ API (include/gavis/gavis_b200.hpp):
// the wall fixture of R/tests/test_planner.cpp:143-161 -- build a field from the
// front view, score {front, back}, expect the unexplored back view.
#include <cstdio>

#include "gavis/gavis_b200.hpp"

using namespace gavis_b200;

int main() {
  Scene scene;
  for (int i = 0; i < 5; ++i)
    for (int j = 0; j < 5; ++j) {
      GaussianParticle g;
      g.position = Vec3(1.0, 0.3 + 0.1 * i, 0.3 + 0.1 * j);
      g.scale = Vec3(0.06, 0.06, 0.06);
      g.opacity = 0.9;
      for (int k = 0; k < 3; ++k) g.color_sh[k] = {0.62 / kY00};
      scene.particles.push_back(g);
    }
  CameraView front = make_lookat(Vec3(0.3, 0.5, 0.5), Vec3(1, 0.5, 0.5), Vec3(0, 0, 1), 64, 64);
  CameraView back = make_lookat(Vec3(1.7, 0.5, 0.5), Vec3(1, 0.5, 0.5), Vec3(0, 0, 1), 64, 64);
  Trajectory traj;
  traj.views = {front};
  try {
    VisibilityField field = construct_field(scene, traj, VmfParams(1.0), 2);
    NbvResult nbv = select_nbv(scene, field, {front, back}, RasterConfig{}, UncertaintyConfig{});
    std::printf("scores %.6f %.6f best %d\n", nbv.scores[0], nbv.scores[1], nbv.best_index);
    bool ok = nbv.best_index == 1 && nbv.scores[1] > nbv.scores[0];
    try {
      select_nbv(scene, field, {}, RasterConfig{}, UncertaintyConfig{});
      ok = false;
    } catch (const ParameterError&) {
    }
    return ok ? 0 : 1;
  } catch (const DeviceError& e) {
    std::printf("device error: %s\n", e.what());
    return 5;
  }
}
