// Planner callers through the C++ front-end with the reference signatures
// (planner.hpp:56-107, :155-184, :284-316). Without arguments only the host
// parts run (sample_candidates, vis_coverage); with "gpu" it also runs two
// steps of run_active_mapping on the device.
#include <cstdio>
#include <cstring>

#include "gavis/gavis_b200.hpp"

using namespace gavis_b200;

int main(int argc, char** argv) {
  Bounds b;
  b.min = Vec3(-1, -1, 0);
  b.max = Vec3(3, 2, 2.5);
  OccluderSet occ;
  OccluderRect wall;
  wall.corner = Vec3(1, -1, 0);
  wall.edge_u = Vec3(0, 3, 0);
  wall.edge_v = Vec3(0, 0, 2.5);
  occ.rectangles.push_back(wall);
  occ.sample_density = 16.0;
  PlannerConfig pc;
  pc.num_candidates = 4;
  pc.steps = 2;
  pc.cam_width = pc.cam_height = 32;
  auto cands = sample_candidates(b, occ, pc, 7);
  for (const auto& c : cands)
    std::printf("cand %.17g %.17g %.17g %.17g\n", c.position[0], c.position[1], c.position[2], c.rotation(0, 0));
  Trajectory t;
  t.views = cands;
  std::printf("coverage %.17g\n", vis_coverage(occ, t));
  if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
    Scene s;
    s.bounds = b;
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 10; ++j) {
        GaussianParticle p;
        p.position = Vec3(1.0, -1.0 + 0.25 * i, 0.1 + 0.25 * j);
        p.scale = Vec3(0.09, 0.09, 0.09);
        p.opacity = 0.9;
        for (int c = 0; c < 3; ++c) p.color_sh[c] = {0.5 / kY00};
        s.particles.push_back(p);
      }
    Trajectory init;
    init.views.push_back(make_lookat(Vec3(0, 0, 1.2), Vec3(1, 0, 1.2), Vec3(0, 0, 1), 32, 32));
    MappingContext ctx;
    ctx.density.rho = 10.0;
    MappingLog log = run_active_mapping(s, occ, init, pc, ctx);
    for (const auto& st : log.steps)
      std::printf("step chosen %d score %.17g coverage %.17g\n", st.chosen_index, st.score, st.vis_coverage);
  }
  return 0;
}
