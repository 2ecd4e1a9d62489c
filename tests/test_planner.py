"""Planner callers of the hot path (planner.hpp): sample_candidates
and vis_coverage (host code in the native library, bit-exact against the oracle
restatement on CPU) and run_active_mapping (device, against an oracle loop)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2605_30342_b200 import api, synth
from paper_2605_30342_b200.model import (K_PI, MappingLog, OccluderRect, OccluderSet, ParameterError,
                                         PlannerConfig, RasterConfig, Scene, UncertaintyConfig, VmfParams,
                                         make_lookat)

BOUNDS = ((-1.0, -1.0, 0.0), (3.0, 2.0, 2.5))


def walls():
    return OccluderSet([
        OccluderRect((1.0, -1.0, 0.0), (0.0, 3.0, 0.0), (0.0, 0.0, 2.5)),            # x = 1 wall
        OccluderRect((-1.0, 0.5, 0.0), (2.0, 0.0, 0.0), (0.0, 0.0, 1.0), opaque=False),  # glass
        OccluderRect((2.0, -1.0, 1.2), (0.0, 1.5, 0.0), (0.8, 0.0, 0.0)),            # shelf
    ], sample_density=16.0)


def same_cams(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert np.array_equal(x.rotation, y.rotation) and np.array_equal(x.position, y.position)
        assert (x.width, x.height, x.fov_h, x.fov_v, x.near) == (y.width, y.height, y.fov_h, y.fov_v, y.near)


@pytest.mark.parametrize("mode,look_inward", [(0, True), (0, False), (1, True)])
@pytest.mark.parametrize("seed", [0, 17, 2 ** 63 + 5])
def test_sample_candidates_bit_exact(mode, look_inward, seed):
    pc = PlannerConfig(mode=mode, look_inward=look_inward, num_candidates=64, clearance=0.25,
                       cam_width=40, cam_height=30, fov_h=1.2, fov_v=0.9, cam_near=0.02)
    got = api.sample_candidates(BOUNDS, walls(), pc, seed)
    ref = O.sample_candidates(BOUNDS, walls(), pc, seed)
    same_cams(got, ref)
    for cam in got:
        R = cam.rotation
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-12)
        if mode == 1:
            assert cam.position[2] == pc.se2_height
        for r in walls().rectangles[::2]:  # opaque ones: clearance respected
            p = np.asarray(cam.position)
            c, u, v = (np.asarray(x, float) for x in (r.corner, r.edge_u, r.edge_v))
            uu = np.clip((p - c) @ u / (u @ u), 0, 1)
            vv = np.clip((p - c) @ v / (v @ v), 0, 1)
            assert np.linalg.norm(c + uu * u + vv * v - p) >= pc.clearance


def test_sample_candidates_deterministic_and_errors():
    pc = PlannerConfig(num_candidates=8)
    a = api.sample_candidates(BOUNDS, None, pc, 3)
    b = api.sample_candidates(BOUNDS, None, pc, 3)
    same_cams(a, b)
    c = api.sample_candidates(BOUNDS, None, pc, 4)
    assert not np.array_equal(a[0].position, c[0].position)
    # look-inward cameras aim at the bounds centre (planner.hpp:89-92)
    ctr = 0.5 * (np.array(BOUNDS[0]) + np.array(BOUNDS[1]))
    for cam in a:
        f = ctr - cam.position
        assert np.allclose(cam.rotation[:, 2], f / np.linalg.norm(f), atol=1e-12)
    with pytest.raises(ParameterError):
        api.sample_candidates(((0, 0, 0), (1, 1, 0)), None, pc, 0)  # zero volume
    with pytest.raises(ParameterError):
        api.sample_candidates(BOUNDS, None, PlannerConfig(num_candidates=0), 0)
    # every position within clearance of a huge opaque wall: budget exhausted
    big = OccluderSet([OccluderRect((-5, -5, 1.25), (10, 0, 0), (0, 10, 0))])
    with pytest.raises(ParameterError, match="budget"):
        api.sample_candidates(BOUNDS, big, PlannerConfig(num_candidates=4, clearance=5.0), 0)


def test_vis_coverage_matches_oracle_and_kat():
    occ = walls()
    cams = api.sample_candidates(BOUNDS, occ, PlannerConfig(num_candidates=6, cam_width=64, cam_height=48), 11)
    for k in range(0, 7):
        assert api.vis_coverage(occ, cams[:k]) == O.vis_coverage(occ, cams[:k])
    assert api.vis_coverage(occ, []) == 0.0
    # test_planner.cpp-style closed case: one wall seen head-on covers it fully
    wall = OccluderSet([OccluderRect((1.0, -0.5, -0.5), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0))])
    cam = make_lookat((0.0, 0.0, 0.0), (1.0, 0.0, 0.0), (0, 0, 1), 64, 64)
    assert api.vis_coverage(wall, [cam]) == 1.0
    back = make_lookat((3.0, 0.0, 0.0), (4.0, 0.0, 0.0), (0, 0, 1), 64, 64)
    assert api.vis_coverage(wall, [back]) == 0.0


# ------------------------------------------------------------------ device
@pytest.fixture(scope="module")
def ctx():
    c = api.Context(0)
    c.set_precision("exact")  # fp64 blend: tolerances at rounding level
    yield c
    c.close()


def room_scene():
    """Wall of opaque splats at x = 1 plus clutter, inside BOUNDS."""
    parts = []
    for i in range(12):
        for j in range(10):
            parts.append(synth.make_particle((1.0, -1.0 + 0.25 * i, 0.1 + 0.25 * j), 0.09, 0.9, (0.6, 0.5, 0.4)))
    g = synth.SplitMix64(5)
    for _ in range(150):
        p = (g.uniform(-0.8, 2.8), g.uniform(-0.8, 1.8), g.uniform(0.1, 2.3))
        parts.append(synth.make_particle(p, g.uniform(0.02, 0.08), g.uniform(0.2, 0.9),
                                         (g.uniform(0, 1), g.uniform(0, 1), g.uniform(0, 1))))
    return Scene.from_particles(parts, 0, bounds=BOUNDS)


def augmented(scene, kept, seed, rho, eta):
    """The device's augmented scene: real particles, then the kept probes in sampling
    order (fp32 positions/scale, identity rotation, o = 0, virtual)."""
    bmin, bmax = np.array(BOUNDS[0]), np.array(BOUNDS[1])
    sc = np.float32(math.cbrt(3.0 * (1.0 + eta) / (4.0 * K_PI * rho)))
    probes = []
    for k in kept:
        g = synth.SplitMix64(synth.derive_seed(seed, int(k)))
        u = (g.next_double(), g.next_double(), g.next_double())
        pos = [np.float32(bmin[d] + (bmax[d] - bmin[d]) * u[d]) for d in range(3)]
        probes.append(dict(pos=pos, scale=float(sc), opacity=0.0, virtual=True))
    ps = Scene.from_particles(probes, scene.color_degree, bounds=BOUNDS)
    cat = lambda a, b: np.concatenate([a, b], 0)
    return Scene(cat(scene.positions, ps.positions), cat(scene.rotations, ps.rotations), cat(scene.scales, ps.scales),
                 cat(scene.opacities, ps.opacities), cat(scene.colors, ps.colors),
                 cat(scene.is_virtual, ps.is_virtual), scene.color_degree, scene.bounds_min, scene.bounds_max)


def oracle_active_mapping(scene, occ, init, pc, rc, uc, rho, eta, eps_v, dseed, density_enabled):
    traj, out = list(init), []
    for step in range(pc.steps):
        aug = scene
        if density_enabled:
            s = O.derive_seed(dseed, step)
            kept, _ = O.density_control(scene, BOUNDS[0], BOUNDS[1], traj, rho=rho, eta=eta, eps_v=eps_v,
                                        seed=s, rc=rc, round_f32=True)
            aug = augmented(scene, kept, s, rho, eta)
        osc = O.OracleScene(aug)
        gamma = O.construct_field(osc, traj, 1.0, 2, rc, threads=8)
        cands = O.sample_candidates(BOUNDS, occ, pc, O.derive_seed(pc.seed, step))
        best, scores = O.select_nbv(osc, gamma, 2, len(traj), cands, rc, uc, threads=8)
        traj.append(cands[best])
        out.append((best, scores, O.vis_coverage(occ, traj)))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("density_enabled", [False, True])
def test_active_mapping_matches_oracle(ctx, density_enabled):
    scene = room_scene()
    occ = walls()
    rc, uc = RasterConfig(), UncertaintyConfig()
    init = [make_lookat((0.0, 0.0, 1.2), (1.0, 0.0, 1.2), (0, 0, 1), 48, 48)]
    pc = PlannerConfig(num_candidates=12, steps=3, seed=21, cam_width=48, cam_height=48, clearance=0.15)
    dc = api.DensityControlConfig(rho=20.0, eta=0.5, eps_v=0.95, seed=9)
    log = api.active_mapping(ctx, scene, occ, init, pc, VmfParams(1.0), 2, rc, uc, dc, density_enabled,
                             bounds=BOUNDS)
    assert isinstance(log, MappingLog) and len(log.steps) == 3
    ref = oracle_active_mapping(scene, occ, init, pc, rc, uc, 20.0, 0.5, 0.95, 9, density_enabled)
    for st, (best, scores, cov) in zip(log.steps, ref):
        assert st.chosen_index == best
        assert np.max(np.abs(st.scores - scores) / np.maximum(1.0, np.abs(scores))) <= 1e-12
        assert st.score == st.scores[best] and st.vis_coverage == cov
        assert st.mean_entropy == st.score / (48 * 48)
    cands0 = api.sample_candidates(BOUNDS, occ, pc, O.derive_seed(pc.seed, 0))
    same_cams([log.chosen_views[0]], [cands0[log.steps[0].chosen_index]])


@pytest.mark.gpu
def test_active_mapping_errors(ctx):
    scene = room_scene()
    with pytest.raises(ParameterError):
        api.active_mapping(ctx, scene, None, [], PlannerConfig(steps=1), bounds=BOUNDS)
    with pytest.raises(ParameterError):
        api.active_mapping(ctx, scene, None, [synth.z_camera()], PlannerConfig(num_candidates=0), bounds=BOUNDS)
    log = api.active_mapping(ctx, scene, None, [synth.z_camera()], PlannerConfig(steps=0), bounds=BOUNDS)
    assert log.steps == [] and log.chosen_views == []


# ---- against the reference ITSELF (oracle/_ref: its unmodified planner.hpp /
# vfield.hpp compiled against the Eigen-subset shim) ---------------------------
def _ref():
    import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R


@pytest.mark.parametrize("mode,look_inward", [(0, True), (0, False), (1, True)])
def test_sample_candidates_equal_the_reference(mode, look_inward):
    R = _ref()
    pc = PlannerConfig(mode=mode, look_inward=look_inward, num_candidates=48, clearance=0.25,
                       cam_width=40, cam_height=30, fov_h=1.2, fov_v=0.9, cam_near=0.02)
    for seed in (0, 17, 2 ** 63 + 5):
        same_cams(api.sample_candidates(BOUNDS, walls(), pc, seed), R.sample_candidates(BOUNDS, walls(), pc, seed))


def test_vis_coverage_equals_the_reference():
    R = _ref()
    pc = PlannerConfig(num_candidates=12, clearance=0.25)
    views = api.sample_candidates(BOUNDS, walls(), pc, 5)
    for k in (0, 1, 4, 12):
        assert api.vis_coverage(walls(), views[:k]) == R.vis_coverage(walls(), views[:k])


def _probe_positions(seed, ks, bmin, bmax):
    """The reference's probe k position (vfield.hpp:172-178): SplitMix64 seeded with
    derive_seed(seed, k), three next_double draws, min + extent * u."""
    M = (1 << 64) - 1
    bmin, bmax = np.asarray(bmin, np.float64), np.asarray(bmax, np.float64)
    out = []
    for k in ks:
        st = O.derive_seed(seed, int(k))
        u = []
        for _ in range(3):
            st = (st + 0x9E3779B97F4A7C15) & M
            z = st
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
            z = z ^ (z >> 31)
            u.append(float(z >> 11) * 2.0 ** -53)
        out.append(bmin + (bmax - bmin) * np.array(u))
    return np.array(out).reshape(-1, 3)


def test_density_control_equals_the_reference():
    """The restatement's kept probes (fp64 probes, round_f32 off) are the
    reference's, probe for probe; the device keeps the same set up to its fp32
    storage of the probes (test_density_control.py)."""
    R = _ref()
    sc = room_scene()
    cams = [make_lookat((0.0, 0.0, 1.2), (1.0, 0.0, 1.2), (0, 0, 1), 48, 48),
            make_lookat((2.5, 1.5, 1.8), (0.0, 0.0, 0.5), (0, 0, 1), 40, 32)]
    for seed, rho in ((9, 20.0), (3, 35.0)):
        kept, _ = O.density_control(sc, BOUNDS[0], BOUNDS[1], cams, rho=rho, eta=0.5, eps_v=0.95, seed=seed,
                                    round_f32=False)
        pos = R.density_control_positions(sc, BOUNDS[0], BOUNDS[1], cams, rho=rho, eta=0.5, eps_v=0.95,
                                          seed=seed, threads=4)
        assert len(kept) == len(pos) > 0
        assert np.array_equal(_probe_positions(seed, kept, BOUNDS[0], BOUNDS[1]), pos)


@pytest.mark.gpu
@pytest.mark.parametrize("density_enabled", [False, True])
def test_active_mapping_matches_the_reference(ctx, density_enabled):
    """The device's run_active_mapping (gavis_active_mapping: density control, field
    rebuild, candidate sampling, select_nbv per step) against the reference's own
    run_active_mapping (planner.hpp:284-316): chosen candidates, their scores and
    coverage per step."""
    R = _ref()
    scene = room_scene()
    occ = walls()
    rc, uc = RasterConfig(), UncertaintyConfig()
    init = [make_lookat((0.0, 0.0, 1.2), (1.0, 0.0, 1.2), (0, 0, 1), 48, 48)]
    pc = PlannerConfig(num_candidates=12, steps=3, seed=21, cam_width=48, cam_height=48, clearance=0.15)
    dc = api.DensityControlConfig(rho=20.0, eta=0.5, eps_v=0.95, seed=9)
    log = api.active_mapping(ctx, scene, occ, init, pc, VmfParams(1.0), 2, rc, uc, dc, density_enabled,
                             bounds=BOUNDS)
    ref = R.active_mapping(scene, BOUNDS, occ, init, pc, 1.0, 2, rc, uc, density_enabled, rho=20.0, eta=0.5,
                           eps_v=0.95, dseed=9, threads=4)
    for st, (best, scores, cov) in zip(log.steps, ref):
        assert st.chosen_index == best
        assert np.max(np.abs(st.scores - scores) / np.maximum(1.0, np.abs(scores))) <= 1e-9
        assert st.vis_coverage == cov
