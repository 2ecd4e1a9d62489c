"""Pin the CPU oracle against every known-answer test the reference suite holds for
the hot path. Scenes are built in double here, exactly like the
reference tests build them, so the reference's own tolerances apply unchanged.

Each test cites the reference test it restates (R/ = /root/reference/proj/).
"""
import math

import numpy as np
import pytest

import oracle as O
from paper_2605_30342_b200.model import (K_GAUSS_ENTROPY, K_PI, K_Y00, RasterConfig, Scene,
                                         UncertaintyConfig, make_lookat, fibonacci_sphere)
from paper_2605_30342_b200 import synth

F64 = np.float64
RC = RasterConfig()


def particle(pos, scale, opacity, color):
    return synth.make_particle(pos, scale, opacity, color)


def scene_of(parts, bounds=None):
    return Scene.from_particles(parts, 0, bounds=bounds, dtype=F64)


def z_cam(w=64, h=64):
    return synth.z_camera(w, h)


# ------------------------------------------------------------------ sh.hpp
def test_sh_constant_and_axis_values():
    """R/tests/test_sh.cpp:40-47"""
    for d in ([0, 0, 1], [1, 0, 0], [0.6, 0.0, 0.8]):
        assert abs(O.eval_sh(0, d)[0] - 0.28209479177387814) <= 1e-15
    assert abs(O.eval_sh(1, [0, 0, 1])[2] - 0.4886025119029199) <= 1e-14
    assert abs(O.eval_sh(1, [0, 0, -1])[2] + 0.4886025119029199) <= 1e-14


def test_sh_sum_rule_and_no_condon_shortley():
    """test_sh.cpp:49-62 sum rule; sh.hpp:30-37 flat index 1,2,3 = c*(y,z,x)."""
    for d in fibonacci_sphere(17):
        b = O.eval_sh(5, d)
        for l in range(6):
            s = sum(b[l * l + l + m] ** 2 for m in range(-l, l + 1))
            assert abs(s - (2 * l + 1) / (4 * K_PI)) <= 1e-10
    d = np.array([0.3, -0.5, 0.8]) / np.linalg.norm([0.3, -0.5, 0.8])
    b = O.eval_sh(1, d)
    c = 0.4886025119029199
    assert np.allclose(b[1:4], c * np.array([d[1], d[2], d[0]]), atol=1e-15)


def test_bessel_and_vmf_scales():
    """sh.hpp:140-147; kappa=1 -> [5.43285, 1.70067, 0.330829, 0.04653];
    test_sh.cpp:150-157 kappa=0 expansion -> 4*pi*Y00 = 3.5449077018110318."""
    s = O.vmf_scales(1.0, 3)
    assert np.allclose(s, [5.43285, 1.70067, 0.330829, 0.04653], rtol=2e-5)
    s0 = O.vmf_scales(0.0, 4)
    assert abs(s0[0] * K_Y00 - 3.5449077018110318) < 1e-14 and np.all(s0[1:] == 0.0)
    assert abs(4 * K_PI * K_Y00 - 3.5449077018110318) < 1e-14
    assert abs(O.bessel_i(0, 1.0) - math.sinh(1.0)) < 1e-15


# -------------------------------------------------------------- raster.hpp
def test_empty_scene_renders_black():
    """test_raster.cpp:104-110"""
    rgb, depth, T = O.rasterize(Scene.empty(), z_cam(), RC)
    assert np.all(rgb == 0) and np.all(depth == 0) and np.all(T == 1)


def test_single_opaque_splat():
    """test_raster.cpp:112-123: clamped alpha 0.99 at the center pixel."""
    cam = make_lookat((0, 0, 0), (0, 0, 1), (0, 1, 0), 129, 129)
    sc = scene_of([particle((0, 0, 1), 1.0, 1.0, (0.5, 0.5, 0.5))])
    rgb, depth, T = O.rasterize(sc, cam, RC)
    pix = 64 * 129 + 64
    assert abs(rgb[pix * 3] - 0.99 * 0.5) <= 1e-12
    assert abs(rgb[pix * 3 + 1] - 0.99 * 0.5) <= 1e-12
    assert abs(T[pix] - 0.01) <= 1e-12
    assert abs(depth[pix] - 0.99) <= 1e-12


def test_colocated_index_tie_break():
    """test_raster.cpp:125-141"""
    cam = make_lookat((0, 0, 0), (0, 0, 1), (0, 1, 0), 129, 129)
    a = particle((0, 0, 1), 1.0, 0.5, (1, 0, 0))
    b = particle((0, 0, 1), 1.0, 0.5, (0, 0, 1))
    pix = 64 * 129 + 64
    rgb, _, T = O.rasterize(scene_of([a, b]), cam, RC)
    assert abs(rgb[pix * 3] - 0.5) <= 1e-12 and abs(rgb[pix * 3 + 2] - 0.25) <= 1e-12
    assert abs(T[pix] - 0.25) <= 1e-12
    rgb, _, _ = O.rasterize(scene_of([b, a]), cam, RC)
    assert abs(rgb[pix * 3 + 2] - 0.5) <= 1e-12 and abs(rgb[pix * 3] - 0.25) <= 1e-12


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_weights_and_transmittance_sum_to_one(seed):
    """test_raster.cpp:143-154 (white scenes: red channel = weight sum)."""
    sc = synth.random_scene(seed, 100, white=True, dtype=F64)
    rgb, _, T = O.rasterize(sc, z_cam(), RC)
    assert np.max(np.abs(rgb[0::3] + T - 1.0)) < 1e-5


def test_acceptance_saturated_white_conservation():
    """acceptance_main.cpp:232-240: derive_seed(0xc0, s), 128^2, saturated white."""
    cam = make_lookat((0, 0, 0), (0, 0, 1), (0, 1, 0), 128, 128)
    for s in range(4):
        sc = synth.random_scene(synth.derive_seed(0xC0, s), 100, white=True, white_value=1.5, dtype=F64)
        rgb, _, T = O.rasterize(sc, cam, RC)
        assert np.max(np.abs(rgb[0::3] + T - 1.0)) < 1e-5


@pytest.mark.parametrize("tile", [16, 5, 13])
def test_tiled_matches_brute_force(tile):
    """test_raster.cpp:156-173; acceptance_main.cpp:242-256 (tile 13)."""
    sc = synth.random_scene(21, 100, dtype=F64)
    rc = RasterConfig(tile_size=tile)
    a = O.rasterize(sc, z_cam(), rc)
    b = O.rasterize_brute(sc, z_cam(), rc)
    for x, y in zip(a, b):
        assert np.max(np.abs(x - y)) < 1e-6


def test_storage_order_invariance():
    """test_raster.cpp:175-187"""
    sc = synth.random_scene(31, 80, dtype=F64)
    rev = sc.subset(slice(None, None, -1))
    a = O.rasterize(sc, z_cam(), RC)
    b = O.rasterize(rev, z_cam(), RC)
    assert np.max(np.abs(a[0] - b[0])) < 1e-6 and np.max(np.abs(a[2] - b[2])) < 1e-6


def test_binning_touched_tiles():
    """test_raster.cpp:202-220"""
    tiny = O.Splat(0, 0, 24.5, 24.5, 0, 0, 0, 1.0, 0.4, 1.0)
    wide = O.Splat(1, 0, 32.0, 32.0, 0, 0, 0, 1.0, 200.0, 1.0)
    off, ent = O.splat_binning([tiny, wide], 64, 64, 16)
    assert len(off) == 17
    for ty in range(4):
        for tx in range(4):
            lst = ent[off[ty * 4 + tx]: off[ty * 4 + tx + 1]]
            assert (0 in lst) == (tx == 1 and ty == 1)
            assert 1 in lst


def test_covered_pixel_range():
    """test_raster.cpp:222-232"""
    assert O.covered_pixel_range(5.0, 1.0, 100) == (4, 5)
    lo, hi = O.covered_pixel_range(0.2, 0.05, 100)
    assert lo > hi
    lo, hi = O.covered_pixel_range(-3.0, 1.0, 100)
    assert lo == 0 and hi < lo


def test_single_view_visibility_unoccluded_is_one():
    """test_raster.cpp:234-240"""
    sc = scene_of([particle((0, 0, 2), 0.05, 0.7, (1, 1, 1))])
    v = O.single_view_visibility(sc, z_cam(), RC)
    assert v[0] == 1.0


def test_single_view_visibility_outside_frustum_is_zero():
    """test_raster.cpp:242-249"""
    sc = scene_of([particle((0, 0, -2), 0.05, 0.7, (1, 1, 1)), particle((40, 0, 2), 0.05, 0.7, (1, 1, 1))])
    v = O.single_view_visibility(sc, z_cam(), RC)
    assert v[0] == 0.0 and v[1] == 0.0


def test_single_view_visibility_behind_blocker():
    """test_raster.cpp:251-263 (+ ray-march oracle, oracle.hpp:70-103)."""
    cam = make_lookat((0, 0, 0), (1, 0, 0), (0, 0, 1), 129, 129)
    sc = scene_of([particle((1, 0, 0), 0.75, 1.0, (1, 1, 1)), particle((2, 0, 0), 0.02, 0.5, (1, 1, 1))])
    v = O.single_view_visibility(sc, cam, RC)
    assert v[0] == 1.0
    assert abs(v[1] - 0.01) <= 1e-3
    t = O.raymarch_transmittance(sc, cam.position, [2, 0, 0], 1e-3, 1)
    assert abs(v[1] - t) < 1e-3


def test_occluder_never_raises_visibility():
    """test_raster.cpp:265-277"""
    bare = [particle((0.2, -0.1, 4), 0.15, 0.8, (1, 1, 1))]
    vb = O.single_view_visibility(scene_of(bare), z_cam(), RC)
    blocked = bare + [particle((0.2, y, 2), 0.25, 0.6, (1, 1, 1)) for y in (-0.3, 0.0, 0.3)]
    vk = O.single_view_visibility(scene_of(blocked), z_cam(), RC)
    assert vk[0] <= vb[0] + 1e-12 and vk[0] < vb[0]


def test_wall_target_matches_raymarch():
    """acceptance_main.cpp:258-283 / gavis_main.cpp:226-257: 9x9 wall + target, <= 5e-2."""
    parts = []
    for i in range(-4, 5):
        for j in range(-4, 5):
            parts.append(dict(pos=(1.0, 0.15 * i, 0.15 * j), scale=0.1, opacity=0.9, color_sh=[[2.0]] * 3))
    parts.append(dict(pos=(1.6, 0.0, 0.0), scale=0.02, opacity=0.5, color_sh=[[2.0]] * 3))
    sc = scene_of(parts)
    cam = make_lookat((0, 0, 0), (1, 0, 0))
    v = O.single_view_visibility(sc, cam, RC)
    t = O.raymarch_transmittance(sc, cam.position, [1.6, 0, 0], 1e-3, len(parts) - 1)
    assert abs(v[-1] - t) <= 5e-2


# -------------------------------------------------------------- vfield.hpp
def opaque(pos, scale, opacity):
    return dict(pos=pos, scale=scale, opacity=opacity, color_sh=[[0.62 / K_Y00]] * 3)


def test_field_rows_zero_for_unobserved_and_virtual():
    """test_vfield.cpp:56-71"""
    parts = [opaque((-5, 0, 0), 0.05, 0.8), dict(opaque((1, 0, 0), 0.05, 0.0), virtual=True)]
    sc = scene_of(parts)
    view = make_lookat((0, 0, 0), (1, 0, 0))
    g = O.construct_field(sc, [view], 1.0, 2, RC)
    assert g.shape == (2, 9) and np.all(g == 0.0)
    assert O.query_visibility(g[0], 2, 1, False, [1, 0, 0]) == 0.0
    assert O.query_visibility(g[1], 2, 1, True, [1, 0, 0]) == 0.0


def test_isotropic_single_view_constant_band():
    """test_vfield.cpp:73-89"""
    sc = scene_of([opaque((1, 0, 0), 0.05, 0.8)])
    g = O.construct_field(sc, [make_lookat((0, 0, 0), (1, 0, 0))], 0.0, 2, RC)
    assert abs(g[0, 0] - 4.0 * K_PI * K_Y00) <= 1e-12 * abs(g[0, 0])
    assert np.all(g[0, 1:] == 0.0)
    assert abs(O.query_visibility(g[0], 2, 1, False, [1, 0, 0]) - 1.0) <= 1e-12
    assert abs(O.query_visibility(g[0], 2, 1, False, [0, 0, 1]) - 1.0) <= 1e-12


def test_repeated_view_doubles_exactly_and_additivity():
    """test_vfield.cpp:91-131"""
    sc = synth.wall_scene(F64)
    v0 = make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5))
    v1 = make_lookat((0.4, 0.3, 0.6), (1, 0.5, 0.5))
    v2 = make_lookat((0.5, 0.7, 0.4), (1, 0.4, 0.5))
    f1 = O.construct_field(sc, [v0], 1.0, 2, RC)
    f2 = O.construct_field(sc, [v0, v0], 1.0, 2, RC)
    assert np.array_equal(f2, 2.0 * f1)
    whole = O.construct_field(sc, [v0, v1, v2], 1.0, 2, RC)
    a = O.construct_field(sc, [v0, v1], 1.0, 2, RC)
    b = O.construct_field(sc, [v2], 1.0, 2, RC)
    assert np.array_equal(whole, a + b)
    c = O.construct_field(sc, [v0], 1.0, 2, RC)
    d = O.construct_field(sc, [v1, v2], 1.0, 2, RC)
    assert np.max(np.abs(whole - (c + d))) <= 1e-12


def test_thread_count_bit_identity():
    """test_vfield.cpp:133-141; planner 163-180 (threads 1 vs 4)."""
    sc = synth.wall_scene(F64)
    views = [make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5)), make_lookat((0.4, 0.4, 0.4), (1, 0.5, 0.5))]
    assert np.array_equal(O.construct_field(sc, views, 1.0, 2, RC, 1), O.construct_field(sc, views, 1.0, 2, RC, 4))


def test_four_view_closed_form_and_amgm():
    """test_vfield.cpp:167-200: kappa=0, 4 x v=0.3 -> 0.7599; AM-GM bound (seed 20240817)."""
    sc = scene_of([opaque((1, 0, 0), 0.05, 0.8)])
    view = make_lookat((0, 0, 0), (1, 0, 0))
    g = np.zeros(9)
    for _ in range(4):
        O.accumulate_view(g, 2, 0.0, sc, view, [0.3])
    v = O.query_visibility(g, 2, 4, False, [0, 1, 0])
    assert abs(v - 0.7599) <= 1e-9
    assert abs(v - (1 - 0.7 ** 4)) <= 1e-12
    rng = synth.SplitMix64(20240817)
    for trial in range(1000):
        n = 1 + rng.next_below(8)
        equal = trial % 5 == 0
        shared = rng.next_double()
        b = [shared if equal else rng.next_double() for _ in range(n)]
        g = np.zeros(9)
        for bi in b:
            O.accumulate_view(g, 2, 0.0, sc, view, [bi])
        est = O.query_visibility(g, 2, n, False, [0, 0, 1])
        exact = 1.0 - np.prod([1.0 - x for x in b])
        assert est <= exact + 1e-12
        if equal:
            assert abs(est - exact) <= 1e-12


def test_mean_estimator_non_monotone():
    """test_vfield.cpp:202-219"""
    sc = scene_of([opaque((1, 0, 0), 0.05, 0.8)])
    view = make_lookat((0, 0, 0), (1, 0, 0))
    one = np.zeros(9)
    O.accumulate_view(one, 2, 0.0, sc, view, [0.9])
    assert abs(O.query_visibility(one, 2, 1, False, [1, 0, 0]) - 0.9) <= 1e-12
    two = np.zeros(9)
    O.accumulate_view(two, 2, 0.0, sc, view, [0.9])
    O.accumulate_view(two, 2, 0.0, sc, view, [0.1])
    assert abs(O.query_visibility(two, 2, 2, False, [1, 0, 0]) - 0.75) <= 1e-12


def test_view_query_at_training_pose():
    """test_vfield.cpp:221-237"""
    sc = synth.wall_scene(F64)
    sc = Scene.from_particles([dict(pos=tuple(p), scale=0.06, opacity=0.9, color_sh=[[0.62 / K_Y00]] * 3)
                               for p in sc.positions] + [opaque((1.3, 0.5, 0.5), 0.04, 0.7)], 0, dtype=F64)
    view = make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5))
    b = O.single_view_visibility(sc, view, RC)
    g = O.construct_field(sc, [view], 0.0, 2, RC)
    idx, vis = O.query_view(g, 2, 1, sc, view)
    assert len(idx) > 0
    for k, i in enumerate(idx):
        assert abs(vis[k] - b[i]) <= 1e-9


def test_view_query_culls():
    """test_vfield.cpp:239-254"""
    sc = scene_of([opaque((1, 0, 0), 0.05, 0.8), opaque((-3, 0, 0), 0.05, 0.5)])
    view = make_lookat((0, 0, 0), (1, 0, 0))
    g = O.construct_field(sc, [view], 1.0, 2, RC)
    idx, _ = O.query_view(g, 2, 1, sc, view)
    assert list(idx) == [0]
    idx, _ = O.query_view(g, 2, 1, sc, make_lookat((5, 0, 0), (6, 0, 0)))
    assert len(idx) == 0


def test_anisotropic_drop_behind_wall():
    """test_vfield.cpp:256-283"""
    sc = synth.wall_scene(F64)
    front = make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5))
    back = make_lookat((1.7, 0.5, 0.5), (1, 0.5, 0.5))
    g = O.construct_field(sc, [front], 1.0, 2, RC)
    _, qf = O.query_view(g, 2, 1, sc, front)
    _, qb = O.query_view(g, 2, 1, sc, back)
    assert len(qf) == 25 and len(qb) == 25
    assert qf.mean() > 0.5 and qb.mean() < 0.5 * qf.mean()
    gi = O.construct_field(sc, [front], 0.0, 2, RC)
    _, a = O.query_view(gi, 2, 1, sc, front)
    _, b = O.query_view(gi, 2, 1, sc, back)
    assert np.max(np.abs(a - b)) <= 1e-9


# --------------------------------------------------------- uncertainty.hpp
EXACT_CAM = make_lookat((0, 0, 0), (0, 0, 1), (0, 1, 0), 129, 129)
EXACT_RC = RasterConfig(alpha_clamp_max=1.0)
CENTER = 64 * 129 + 64


def exact_scene():
    """test_uncertainty.cpp:47-59 ExactFixture"""
    return Scene.from_particles([dict(pos=(0, 0, 1), scale=0.01, opacity=1.0, color_sh=[[0.5 / K_Y00]] * 3)],
                                0, bounds=((-1, -1, 0), (1, 1, 2)), dtype=F64)


def test_fully_visible_unit_alpha_pixel():
    """test_uncertainty.cpp:125-144"""
    sc = exact_scene()
    g = O.construct_field(sc, [EXACT_CAM], 0.0, 2, EXACT_RC)
    uc = UncertaintyConfig(color_sigma=1.0)
    H, w0, depth = O.render_entropy(sc, g, 2, 1, EXACT_CAM, EXACT_RC, uc)
    assert abs(H[CENTER] - K_GAUSS_ENTROPY) <= 1e-12
    assert abs(w0[CENTER]) <= 1e-12
    assert abs(depth[CENTER] - 1.0) <= 1e-12
    assert H[0] == 0.0 and w0[0] == 0.0 and depth[0] == 0.0


def test_hidden_splat_routes_through_prior():
    """test_uncertainty.cpp:146-171"""
    sc = exact_scene()
    uc = UncertaintyConfig(color_sigma=0.1)
    H, w0, _ = O.render_entropy_core(sc, EXACT_CAM, EXACT_RC, uc, [0.0])
    assert abs(w0[CENTER] - 0.575) <= 1e-12
    assert abs(H[CENTER] - w0[CENTER] * (-math.log(w0[CENTER]) + K_GAUSS_ENTROPY)) <= 1e-12
    Hs, w0s, _ = O.render_entropy_core(sc, EXACT_CAM, EXACT_RC, uc, [1.0])
    assert Hs[CENTER] < 0.0 and H[CENTER] > Hs[CENTER] and w0s[CENTER] == 0.0


def test_beta_one_reduces_to_rasterize():
    """test_uncertainty.cpp:173-197 (transmittance / depth part; colour via mixtures is
    out of scope): with beta=1 the compensated alpha is the plain alpha."""
    sc = synth.random_scene(0xCA4D1D, 40, dtype=F64)
    cam = z_cam()
    vis = np.array([synth.SplitMix64(17).next_double() for _ in range(1)] * sc.num_particles)
    uc = UncertaintyConfig(beta=1.0, color_sigma=0.3)
    H, w0, depth = O.render_entropy_core(sc, cam, RC, uc, vis)
    _, rdepth, _ = O.rasterize(sc, cam, RC)
    assert np.max(np.abs(depth - rdepth)) <= 1e-9


def test_mass_conservation_and_full_visibility():
    """test_uncertainty.cpp:199-217 (sum w v + w0 + T = 1) and :255-264 (v = 1 -> w0 = 0).
    With v constant per pixel the seen mass is (1 - T - w0) * 1 when v==1."""
    sc = synth.random_scene(0xACE, 30, dtype=F64)
    cam = z_cam()
    _, w0, _ = O.render_entropy_core(sc, cam, RC, UncertaintyConfig(), np.ones(30))
    assert np.all(w0 == 0.0)
    # v == 0 everywhere: all composited mass is invisible, so w0 + T = 1 with T from the
    # compensated track; compare against T computed from the alpha*-only rasterization.
    _, w0z, _ = O.render_entropy_core(sc, cam, RC, UncertaintyConfig(), np.zeros(30))
    assert np.all(w0z >= 0.0) and np.all(w0z <= 1.0)


def test_image_entropy_sum():
    """test_uncertainty.cpp:345-358"""
    assert abs(O.image_entropy([1.0, 2.0]) - 3.0) <= 1e-15
    assert O.image_entropy([0.0, 0.0]) == 0.0


def test_field_driven_maps_finite_bounded():
    """test_uncertainty.cpp:390-416"""
    sc = synth.random_scene(0xF00D, 80, dtype=F64)
    train = z_cam()
    query = make_lookat((0.5, 0.3, 0.2), (0, 0, 4), (0, 1, 0), 64, 64)
    g = O.construct_field(sc, [train], 1.0, 2, RC)
    uc = UncertaintyConfig(color_sigma=1.0)
    H, w0, _ = O.render_entropy(sc, g, 2, 1, query, RC, uc)
    assert np.all(np.isfinite(H)) and np.all(H >= 0) and np.all(w0 >= 0) and np.all(w0 <= 1)
    assert H.sum() > 0


# ------------------------------------------------------------- planner.hpp
def test_select_nbv_prefers_unexplored_and_ties_low_index():
    """test_planner.cpp:143-180"""
    sc = synth.wall_scene(F64)
    front = make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5), (0, 0, 1), 64, 64)
    back = make_lookat((1.7, 0.5, 0.5), (1, 0.5, 0.5), (0, 0, 1), 64, 64)
    g = O.construct_field(sc, [front], 1.0, 2, RC)
    best, scores = O.select_nbv(sc, g, 2, 1, [front, back], RC, UncertaintyConfig())
    assert np.all(np.isfinite(scores)) and scores[1] > scores[0] and best == 1
    best, scores = O.select_nbv(sc, g, 2, 1, [front, front, front], RC, UncertaintyConfig())
    assert best == 0 and scores[1] == scores[0] and scores[2] == scores[0]
    b4, s4 = O.select_nbv(sc, g, 2, 1, [front, front, front], RC, UncertaintyConfig(), threads=4)
    assert b4 == best and np.array_equal(s4, scores)


def test_compensated_alpha_closed_forms():
    """test_uncertainty.cpp:70-92 through a one-splat render: centre alpha = 1 with the
    ExactFixture, so entropy-track alpha* is visible as 1 - T*: v=0 -> 0.575."""
    sc = exact_scene()
    uc = UncertaintyConfig()
    for v, expect in ((1.0, 1.0), (0.0, 0.575)):
        H, w0, depth = O.render_entropy_core(sc, EXACT_CAM, EXACT_RC, uc, [v])
        # depth = w * z with w = alpha* * 1 at the centre, z = 1
        assert abs(depth[CENTER] - expect) <= 1e-12


@pytest.mark.parametrize("provider", [0, 1])
def test_mixture_dump_consistency(provider):
    """render_entropy_core's mixtures_out (uncertainty.hpp:207-230): the components
    reproduce the pixel's entropy, prior weight and residual transmittance
    (sum w* + T* = 1, sum w* (1 - v) = w0) and match the entropy map."""
    sc = synth.random_scene(0x5EED, 40)
    cam = synth.z_camera(48, 40)
    vis = np.array([synth.SplitMix64(99 + i).next_double() for i in range(40)])
    vis[::7] = 0.0
    vis[3::9] = 1.0
    uc = UncertaintyConfig(color_sigma=0.3, variance_provider=provider)
    rc = RasterConfig()
    if provider == 1:
        O.set_coeff_variances(np.full((40, 3, 4), 0.05) + np.arange(40)[:, None, None] * 1e-3, 1)
    try:
        off, comp, prior, resid, H = O.render_mixtures(sc, cam, rc, uc, vis)
        Href, w0ref, _ = O.render_entropy_core(sc, cam, rc, uc, vis)
    finally:
        O.set_coeff_variances(None, -1)
    assert np.array_equal(H, Href) and np.array_equal(prior, w0ref)
    assert off[-1] == len(comp) and off[-1] > 100
    for p in range(cam.width * cam.height):
        c = comp[off[p]:off[p + 1]]
        w, v = c[:, 0], c[:, 1]
        assert np.all(w > 0) and np.all((c[:, 2:5] >= 0) & (c[:, 2:5] <= 1))
        assert abs(w.sum() + resid[p] - 1.0) <= 1e-12
        assert abs((w * (1 - v)).sum() - prior[p]) <= 1e-12
        s = w * v
        hl = 0.5 * np.log(c[:, 5:8]).sum(axis=1)
        h = (s[s > 0] * (-np.log(s[s > 0]) + hl[s > 0] + K_GAUSS_ENTROPY)).sum()
        if prior[p] > 0:
            h += prior[p] * (-math.log(prior[p]) + K_GAUSS_ENTROPY)
        assert abs(h - H[p]) <= 1e-12 * max(1.0, abs(H[p]))
        if provider == 0:
            assert np.all(c[:, 5:8] == 0.09)
