"""The reference ITSELF against the C restatement oracle, on the CPU.

oracle/_ref/libgavis_ref.so is the GAVIS reference's unmodified hot-path headers
(/root/reference/proj/include/gavis/*.hpp) compiled -O3 -ffp-contract=off
against a self-written Eigen-subset shim (oracle/eigen_shim: fixed-size
products summed left to right, Eigen's quaternion-to-matrix formula). Every
hot-path function of the restatement (oracle/gavis_oracle.c), and so the
checker the device is held to, must agree with the reference's own code BIT FOR
BIT: project_scene and splat_binning (raster.hpp:114-164), single_view_visibility
(raster.hpp:237-290), construct_field (vfield.hpp:68-92), rasterize
(raster.hpp:175-231), render_entropy(_core) incl. mixtures and sh_propagation
(uncertainty.hpp:124-260), select_nbv (planner.hpp:117-137); the planner and
density-control rows are pinned in tests/test_planner.py.
"""
import numpy as np
import pytest

import oracle as O
import ref as R
from paper_2605_30342_b200 import synth
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference here)")

UC = UncertaintyConfig()


@pytest.mark.parametrize("tile", [16, 5, 13])
def test_reference_equals_restatement_config1(tile):
    c = synth.config1(0)
    rc = RasterConfig(tile_size=tile)
    osc = O.OracleScene(c["scene"])
    for cam in c["train"][:2]:
        assert np.array_equal(R.single_view_visibility(osc, cam, rc), O.single_view_visibility(osc, cam, rc))
    g_r = R.construct_field(osc, c["train"], 1.0, 2, rc, threads=4)
    g_o = O.construct_field(osc, c["train"], 1.0, 2, rc, threads=4)
    assert np.array_equal(g_r, g_o)
    for cam in c["candidates"][:2]:
        for a, b in zip(R.rasterize(osc, cam, rc), O.rasterize(osc, cam, rc)):
            assert np.array_equal(a, b)
        H_r, w_r, d_r = R.render_entropy(osc, g_r, 2, 16, cam, rc, UC)
        H_o, w_o, d_o = O.render_entropy(osc, g_o, 2, 16, cam, rc, UC)
        assert np.array_equal(H_r, H_o) and np.array_equal(w_r, w_o) and np.array_equal(d_r, d_o)
    b_r, s_r = R.select_nbv(osc, g_r, 2, 16, c["candidates"], rc, UC, threads=4)
    b_o, s_o = O.select_nbv(osc, g_o, 2, 16, c["candidates"], rc, UC, threads=4)
    assert b_r == b_o and np.array_equal(s_r, s_o)


def test_reference_equals_restatement_room_and_hook():
    """Config-3 structure (thin wall slabs: depth ties, flattened conics) and the
    non-default uncertainty paths: correlation hook, beta/o0/sigma variations."""
    c = synth.config3(0, n=60_000, n_train=6, n_candidates=4, res=160)
    rc = RasterConfig()
    osc = O.OracleScene(c["scene"])
    g_r = R.construct_field(osc, c["train"], 1.0, 2, rc, threads=4)
    assert np.array_equal(g_r, O.construct_field(osc, c["train"], 1.0, 2, rc, threads=4))
    for uc in (UC, UncertaintyConfig(beta=0.2, prior_opacity=0.3, color_sigma=0.05),
               UncertaintyConfig(correlation=1, correlation_lambda=2.5)):
        b_r, s_r = R.select_nbv(osc, g_r, 2, 6, c["candidates"], rc, uc, threads=4)
        b_o, s_o = O.select_nbv(osc, g_r, 2, 6, c["candidates"], rc, uc, threads=4)
        assert b_r == b_o and np.array_equal(s_r, s_o)


def test_reference_bench_step_matches_restatement():
    """The reference arm's step (select_nbv + rasterize on a prebuilt scene) scores
    like the restatement."""
    c = synth.config1(3)
    rc = RasterConfig()
    osc = O.OracleScene(c["scene"])
    rs = R.RefScene(osc)
    g = R.construct_field_h(rs, c["train"][:6], 1.0, 2, rc, threads=4)
    b_r, s_r = R.select_nbv_rgb_h(rs, g, 2, 6, c["candidates"][:8], rc, UC, threads=4)
    b_o, s_o = O.select_nbv(osc, g, 2, 6, c["candidates"][:8], rc, UC, threads=4, with_rgb=True)
    assert b_r == b_o and np.array_equal(s_r, s_o)
    rs.close()


def test_reference_mixtures_and_sh_propagation_equal_restatement():
    """render_entropy_core's optional outputs (uncertainty.hpp:124-238): the
    per-pixel mixture dump (components w, v, clamped SH colour, diag Q_c; prior
    weight, residual T, entropy) and the sh_propagation provider (per-splat
    1/2 sum_c ln q_c(d) from coefficient variances), the reference against the
    restatement the device is tested on (tests/test_optional_outputs.py)."""
    c = synth.config1(2)
    sc = c["scene"]
    osc = O.OracleScene(sc)
    rng = np.random.default_rng(4)
    vis = rng.uniform(0.0, 1.0, sc.num_particles)
    cam = c["candidates"][1]
    rc = RasterConfig()
    for uc in (UC, UncertaintyConfig(beta=0.3, prior_opacity=0.2, color_sigma=0.07)):
        (H, w0, d), (off, comps, prior, resid, Hm) = R.render_entropy_core(osc, cam, rc, uc, vis, mixtures=True,
                                                                           threads=4)
        o_off, o_comps, o_prior, o_resid, o_H = O.render_mixtures(osc, cam, rc, uc, vis)
        assert np.array_equal(off, o_off) and np.array_equal(comps, o_comps)
        assert np.array_equal(prior, o_prior) and np.array_equal(resid, o_resid) and np.array_equal(Hm, o_H)
        oH, ow0, od = O.render_entropy_core(osc, cam, rc, uc, vis)
        assert np.array_equal(H, oH) and np.array_equal(w0, ow0) and np.array_equal(d, od)
    var = rng.uniform(0.01, 0.2, size=(sc.num_particles, 3, 9))
    uc = UncertaintyConfig(variance_provider=1)
    H, w0, _ = R.render_entropy_core(osc, cam, rc, uc, vis, coeff_var=var, var_degree=2, threads=4)
    O.set_coeff_variances(var, 2)
    try:
        oH, ow0, _ = O.render_entropy_core(osc, cam, rc, uc, vis)
        (_, _, _), (_, comps, _, _, _) = R.render_entropy_core(osc, cam, rc, uc, vis, coeff_var=var, var_degree=2,
                                                               mixtures=True, threads=4)
        _, o_comps, _, _, _ = O.render_mixtures(osc, cam, rc, uc, vis)
    finally:
        O.set_coeff_variances(None, -1)
    assert np.array_equal(H, oH) and np.array_equal(w0, ow0)
    assert np.array_equal(comps, o_comps)


@pytest.mark.parametrize("tile", [16, 5, 13])
def test_reference_projection_and_binning_equal_restatement(tile):
    """project_scene (raster.hpp:114-130: EWA conics, radii, the (depth, index)
    order) and splat_binning (raster.hpp:145-164: tile lists) of the reference
    against the restatement, field by field -- the restatement the device's keys,
    sorted order and conics are held to bit for bit (test_gpu_parity.py)."""
    for c in (synth.config1(0), synth.config3(0, n=40_000, n_train=2, n_candidates=2, res=128)):
        osc = O.OracleScene(c["scene"])
        for cam in (c["train"][:1] + c["candidates"][:1]):
            sp_r, off_r, ent_r = R.project_and_bin(osc, cam, 0.3, tile)
            sp_o = O.project_scene(osc, cam, 0.3)
            off_o, ent_o = O.splat_binning(sp_o, cam.width, cam.height, tile)
            assert len(sp_r) == len(sp_o) > 0
            for a, b in zip(sp_r, sp_o):
                assert (a.particle_index, a.mean_x, a.mean_y, a.conic_a, a.conic_b, a.conic_c, a.depth, a.radius,
                        a.opacity) == (b.particle_index, b.mean_x, b.mean_y, b.conic_a, b.conic_b, b.conic_c,
                                       b.depth, b.radius, b.opacity)
            assert np.array_equal(off_r, off_o) and np.array_equal(ent_r, ent_o)


def test_reference_query_view_equals_restatement():
    """query_view (vfield.hpp:121-134), the north_star's VF-QUERY entry point:
    indices of the non-culled particles and their AM-GM visibilities."""
    c = synth.config1(0)
    osc = O.OracleScene(c["scene"])
    g = R.construct_field(osc, c["train"][:5], 1.0, 3, RasterConfig(), threads=4)
    for cam in c["candidates"][:3]:
        i_r, v_r = R.query_view(g, 3, 5, osc, cam)
        i_o, v_o = O.query_view(g, 3, 5, osc, cam)
        assert len(i_r) > 0 and np.array_equal(i_r, i_o) and np.array_equal(v_r, v_o)
