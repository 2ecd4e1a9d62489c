"""Non-default uncertainty paths: the sh_propagation variance
provider (uncertainty.hpp:63-83, :149-163) and the correlation hook of the image
score (uncertainty.hpp:273-277, planner.hpp:124-130)."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2605_30342_b200 import synth
from paper_2605_30342_b200.model import ParameterError, RasterConfig, UncertaintyConfig, VmfParams, make_lookat

RC = RasterConfig()


def test_oracle_hook_closed_form():
    """test_uncertainty.cpp:345-371"""
    e, d = [1.0, 2.0], [1.0, 3.0]
    want = 1.0 * (1.0 - math.exp(-0.5)) + 2.0 * (1.0 - math.exp(-1.5))
    assert abs(O.image_entropy_hook(e, d, 2.0) - want) <= 1e-15
    assert abs(O.image_entropy_hook(e, d, 1e-12) - 3.0) <= 1e-12


def test_oracle_propagated_constant_matches_constant_provider():
    """test_uncertainty.cpp:307-329: variance 4 pi sigma^2 on the DC term propagates to sigma^2."""
    sc = synth.random_scene(0xD1CE, 20, dtype=np.float64)
    cam = synth.z_camera()
    vis = np.array([synth.SplitMix64(41 + i).next_double() for i in range(20)])
    ref, _, _ = O.render_entropy_core(sc, cam, RC, UncertaintyConfig(color_sigma=0.2), vis)
    O.set_coeff_variances(np.full((20, 3, 1), 4.0 * math.pi * 0.04), 0)
    got, _, _ = O.render_entropy_core(sc, cam, RC, UncertaintyConfig(variance_provider=1), vis)
    O.set_coeff_variances(None, -1)
    assert np.max(np.abs(got - ref)) <= 1e-9


@pytest.fixture(scope="module")
def ctx():
    from paper_2605_30342_b200 import api
    c = api.Context(0)
    c.set_precision("exact")  # fp64 blend: tolerances at rounding level
    yield c
    c.close()


@pytest.mark.gpu
def test_device_propagation_matches_oracle(ctx):
    from paper_2605_30342_b200 import api
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    rng = np.random.default_rng(7)
    for deg in (0, 2, 3):
        nbv = (deg + 1) ** 2
        var = rng.uniform(0.01, 0.2, size=(scene.num_particles, 3, nbv)).astype(np.float32)
        ds = ctx.upload(scene)
        ds.set_coeff_variances(var, deg)
        f = api.construct_field(ctx, ds, c["train"][:4], VmfParams(1.0), 2, RC)
        g = f.download().gamma
        uc = UncertaintyConfig(variance_provider=1)
        cam = c["candidates"][0]
        r = api.render(ctx, ds, f, [cam], RC, uc, entropy=True, invisible_mass=True, scores=True)
        O.set_coeff_variances(var.astype(np.float64), deg)
        H, w0, _ = O.render_entropy(osc, g, 2, 4, cam, RC, uc)
        O.set_coeff_variances(None, -1)
        assert np.max(np.abs(r["entropy"] - H)) <= 1e-9
        assert np.max(np.abs(r["invisible_mass"] - w0)) <= 1e-12
        assert abs(r["scores"][0] - H.sum()) <= 1e-9 * max(1.0, abs(H.sum()))


@pytest.mark.gpu
def test_device_propagated_constant_equals_constant(ctx):
    from paper_2605_30342_b200 import api
    sc = synth.random_scene(0xD1CE, 20)
    cam = synth.z_camera()
    vis = np.array([synth.SplitMix64(41 + i).next_double() for i in range(20)])
    ref = api.render_entropy_core(ctx, sc, cam, RC, UncertaintyConfig(color_sigma=0.2), vis)
    ds = ctx.upload(sc)
    ds.set_coeff_variances(np.full((20, 3, 1), 4.0 * math.pi * 0.04), 0)
    got = api.render_entropy_core(ctx, ds, cam, RC, UncertaintyConfig(variance_provider=1), vis)
    assert np.max(np.abs(got.entropy - ref.entropy)) <= 1e-6  # fp32-stored variances
    ds.set_coeff_variances(np.zeros((20, 3, 1)), 0)
    with pytest.raises(ParameterError):
        api.render_entropy_core(ctx, ds, cam, RC, UncertaintyConfig(variance_provider=1), vis)
    with pytest.raises(ParameterError):
        api.render_entropy_core(ctx, sc, cam, RC, UncertaintyConfig(variance_provider=1), vis)
    with pytest.raises(ParameterError):
        ds.set_coeff_variances(-np.ones((20, 3, 1)), 0)


@pytest.mark.gpu
def test_device_correlation_hook_scores(ctx):
    from paper_2605_30342_b200 import api
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    f = api.construct_field(ctx, scene, c["train"][:6], VmfParams(1.0), 2, RC)
    g = f.download().gamma
    uc = UncertaintyConfig(correlation=1, correlation_lambda=2.0)
    res = api.select_nbv(ctx, scene, f, c["candidates"][:6], RC, uc)
    best, scores = O.select_nbv(osc, g, 2, 6, c["candidates"][:6], RC, uc, threads=8)
    assert res.best_index == best
    assert np.max(np.abs(res.scores - scores) / np.maximum(1.0, np.abs(scores))) <= 1e-9
    plain = api.select_nbv(ctx, scene, f, c["candidates"][:6], RC, UncertaintyConfig())
    assert np.all(res.scores < plain.scores)


@pytest.mark.gpu
@pytest.mark.parametrize("provider", [0, 1])
def test_device_mixtures_match_oracle(ctx, provider):
    """gavis_ua_mixtures (render_entropy mixtures_out, uncertainty.hpp:207-230)
    against the oracle restatement: CSR offsets bit-exact, components and the
    per-pixel prior weight / residual transmittance / entropy to fp64 rounding."""
    from paper_2605_30342_b200 import api
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    cam = c["candidates"][1]
    rng = np.random.default_rng(3)
    vis = rng.uniform(0, 1, scene.num_particles)
    vis[rng.uniform(size=scene.num_particles) < 0.2] = 0.0
    uc = UncertaintyConfig(variance_provider=provider)
    ds = ctx.upload(scene)
    if provider == 1:
        var = rng.uniform(0.01, 0.2, size=(scene.num_particles, 3, 4)).astype(np.float32)
        ds.set_coeff_variances(var, 1)
        O.set_coeff_variances(var.astype(np.float64), 1)
    try:
        off, comp, prior, resid, H = api.render_mixtures(ctx, ds, None, cam, RC, uc, splat_visibility=vis)
        ooff, ocomp, oprior, oresid, oH = O.render_mixtures(osc, cam, RC, uc, vis)
    finally:
        O.set_coeff_variances(None, -1)
    assert np.array_equal(off, ooff) and off[-1] > 1000
    assert np.max(np.abs(comp[:, :2] - ocomp[:, :2])) <= 1e-12
    assert np.max(np.abs(comp[:, 2:5] - ocomp[:, 2:5])) <= 1e-12
    assert np.max(np.abs(comp[:, 5:] - ocomp[:, 5:]) / ocomp[:, 5:]) <= 1e-12
    assert np.max(np.abs(prior - oprior)) <= 1e-12 and np.max(np.abs(resid - oresid)) <= 1e-12
    assert np.max(np.abs(H - oH)) <= 1e-10
    # consistent with the regular render of the same pixels
    r = api.render(ctx, ds, None, [cam], RC, uc, entropy=True, invisible_mass=True, splat_visibility=vis)
    assert np.max(np.abs(r["entropy"] - H)) <= 1e-10
