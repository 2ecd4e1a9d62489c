"""Certified fp32 UA blend (GAVIS_PRECISION_CERTIFIED, the default) against the CPU
oracle and against the exact fp64 device path.

What the certified path guarantees (kernels_ua_fast.cu header):
  * per-pixel contributor counts of both tracks are bit-exact (uncertified
    early-termination tests are recomputed in fp64);
  * the selected next-best view is the fp64 argmax (candidates within 1e-3 of
    the best are re-scored exactly);
  * RGB / entropy images within the north_star's 1e-4 max-abs (asserted), in
    practice ~1e-6 (asserted at 2e-5), scores within 1e-6 relative.
"""
import numpy as np
import pytest

import oracle as O
from paper_2605_30342_b200 import api, synth
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams, make_lookat

pytestmark = pytest.mark.gpu

RC = RasterConfig()
UC = UncertaintyConfig()
NS_IMAGE_ABS = 1e-4   # north_star: RGB / uncertainty images within 1e-4 max-abs
IMG_ABS = 2e-5        # what the fp32 blend holds on these scenes
SCORE_REL = 1e-6


@pytest.fixture(scope="module")
def ctx():
    c = api.Context(0)
    c.set_precision("certified")
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_exact():
    c = api.Context(0)
    c.set_precision("exact")
    yield c
    c.close()


@pytest.fixture(scope="module")
def room():
    """Config-3 structure (thin wall slabs + clutter) at oracle-friendly size."""
    return synth.config3(0, n=60_000, n_train=12, n_candidates=6, res=160)


def test_certified_rasterize_parity(ctx):
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    for cam in c["candidates"][:3]:
        r = api.render(ctx, scene, None, [cam], RC, UC, rgb=True, depth=True, transmittance=True,
                       contributors=True)
        rgb, depth, T, cc = O.rasterize(osc, cam, RC, contrib=True)
        assert np.array_equal(r["rgb_contributors"], cc)
        assert np.max(np.abs(r["transmittance"] - T)) <= 1e-6
        assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS
        assert np.max(np.abs(r["rgb"] - rgb)) <= NS_IMAGE_ABS
        assert np.max(np.abs(r["depth"] - depth)) <= 1e-4


def _entropy_parity(ctx, scene, train, cams, degree):
    osc = O.OracleScene(scene)
    f = api.construct_field(ctx, scene, train, VmfParams(1.0), degree, RC)
    g = f.download().gamma
    r = api.render(ctx, scene, f, cams, RC, UC, entropy=True, invisible_mass=True, entropy_depth=True,
                   scores=True, contributors=True, rgb=True)
    P = cams[0].width * cams[0].height
    for k, cam in enumerate(cams):
        H, w0, depth, cc = O.render_entropy(osc, g, degree, len(train), cam, RC, UC, contrib=True)
        sl = slice(k * P, (k + 1) * P)
        assert np.array_equal(r["entropy_contributors"][sl], cc)
        assert np.max(np.abs(r["entropy"][sl] - H)) <= IMG_ABS
        assert np.max(np.abs(r["entropy"][sl] - H)) <= NS_IMAGE_ABS
        assert np.max(np.abs(r["invisible_mass"][sl] - w0)) <= 1e-5
        ref = O.image_entropy(H)
        assert abs(r["scores"][k] - ref) <= SCORE_REL * max(1.0, abs(ref))
        rgb, _, _, rc_cc = O.rasterize(osc, cam, RC, contrib=True)
        assert np.array_equal(r["rgb_contributors"][sl], rc_cc)
        assert np.max(np.abs(r["rgb"][3 * k * P:3 * (k + 1) * P] - rgb)) <= IMG_ABS


def test_certified_entropy_parity_config1(ctx):
    c = synth.config1(0)
    _entropy_parity(ctx, c["scene"], c["train"], c["candidates"][:4], 2)


def test_certified_entropy_parity_room(ctx, room):
    _entropy_parity(ctx, room["scene"], room["train"], room["candidates"][:4], 2)


def test_certified_select_nbv_matches_oracle(ctx, room):
    scene = room["scene"]
    f = api.construct_field(ctx, scene, room["train"], VmfParams(1.0), 2, RC)
    g = f.download().gamma
    res = api.select_nbv(ctx, scene, f, room["candidates"], RC, UC)
    best, scores = O.select_nbv(O.OracleScene(scene), g, 2, len(room["train"]), room["candidates"], RC, UC,
                                threads=8)
    assert res.best_index == best
    assert np.max(np.abs(res.scores - scores) / np.maximum(1.0, np.abs(scores))) <= SCORE_REL


def test_certified_argmax_rescoring(ctx):
    """Identical candidates score identically; the tie goes to the lowest index
    after the contenders are re-scored in fp64 (test_planner.cpp:170-180)."""
    c = synth.config1(0)
    scene = c["scene"]
    f = api.construct_field(ctx, scene, c["train"], VmfParams(1.0), 2, RC)
    cam = c["candidates"][5]
    other = c["candidates"][6]
    before = ctx.counters()[1]
    r = api.select_nbv(ctx, scene, f, [cam, cam, cam], RC, UC)
    assert r.best_index == 0 and r.scores[0] == r.scores[1] == r.scores[2]
    assert ctx.counters()[1] - before == 3
    ex = api.select_nbv(ctx, scene, f, [other, cam], RC, UC)
    r = api.select_nbv(ctx, scene, f, [other, cam, cam], RC, UC)
    assert r.best_index == (1 if ex.scores[1] > ex.scores[0] else 0)
    assert r.scores[1] == r.scores[2]


def test_forced_redo_is_exact(ctx, ctx_exact, monkeypatch, room):
    """With every pixel handed to the fp64 redo the certified path must reproduce
    the exact path bit for bit (the redo runs the exact steps) -- except the SH
    colour's dot product: the exact kernel evaluates it on the tensor cores
    (split fp16, fp32 accumulate), the one-warp redo with packed fp32 FMAs, so
    the RGB image agrees to ~1e-7 instead of bit for bit."""
    scene = room["scene"]
    f = api.construct_field(ctx_exact, scene, room["train"], VmfParams(1.0), 2, RC)
    cams = room["candidates"][:2]
    kw = dict(rgb=True, depth=True, transmittance=True, entropy=True, invisible_mass=True,
              entropy_depth=True, scores=True, contributors=True)
    ex = api.render(ctx_exact, scene, f, cams, RC, UC, **kw)
    monkeypatch.setenv("GAVIS_CERT_FORCE_REDO", "1")
    fr = api.render(ctx_exact, scene, f, cams, RC, UC, **kw)  # exact context: knob ignored
    ctx_f = api.Context(0)
    ctx_f.set_precision("certified")
    try:
        fd = api.upload_field(ctx_f, scene, f.download())
        red0 = ctx_f.counters()[0]
        got = api.render(ctx_f, scene, fd, cams, RC, UC, **kw)
        assert ctx_f.counters()[0] - red0 == 2 * cams[0].width * cams[0].height
    finally:
        ctx_f.close()
    assert set(ex) == set(got)
    for k in ex:
        assert np.array_equal(ex[k], fr[k])
        if k == "rgb":
            assert np.max(np.abs(ex[k] - got[k])) <= 2e-6
        else:
            assert np.array_equal(ex[k], got[k]), k


@pytest.mark.parametrize("cfg", [3, 2, 4])
def test_certified_vs_exact_full_size(ctx, ctx_exact, cfg):
    """Configs 3 (1M Gaussians, indoor), 2 (500k, object) at 800^2 and 4 (3M,
    1920x1080) at full size: size-independent agreement of the certified and the
    exact device paths (the exact path is pinned to the oracle)."""
    c = {3: lambda: synth.config3(0, n_candidates=4), 2: lambda: synth.config2(0, n_candidates=4),
         4: lambda: synth.config4(0, n_train=30, n_candidates=4)}[cfg]()
    scene = c["scene"]
    f = api.construct_field(ctx_exact, scene, c["train"][:30], VmfParams(1.0), c["degree"], RC)
    cams = c["candidates"][:4]
    kw = dict(rgb=True, transmittance=True, entropy=True, invisible_mass=True, scores=True, contributors=True)
    ex = api.render(ctx_exact, scene, f, cams, RC, UC, **kw)
    fd = api.upload_field(ctx, scene, f.download())
    got = api.render(ctx, scene, fd, cams, RC, UC, **kw)
    assert np.array_equal(ex["rgb_contributors"], got["rgb_contributors"])
    assert np.array_equal(ex["entropy_contributors"], got["entropy_contributors"])
    assert np.max(np.abs(ex["rgb"] - got["rgb"])) <= IMG_ABS
    assert np.max(np.abs(ex["entropy"] - got["entropy"])) <= IMG_ABS
    assert np.max(np.abs(ex["transmittance"] - got["transmittance"])) <= 1e-6
    assert np.max(np.abs(ex["scores"] - got["scores"]) / np.abs(ex["scores"])) <= 1e-5


def test_certified_variants_match_oracle(ctx):
    """Every instantiation the certified path selects -- entropy only, RGB only,
    extra outputs (depths, counts), the correlation hook, sh_propagation -- and
    the configurations it hands to the exact kernels (tile 13, alpha_clamp_max 1)."""
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    f = api.construct_field(ctx, scene, c["train"], VmfParams(1.0), 2, RC)
    g = f.download().gamma
    cam = c["candidates"][2]
    H, w0, edep, cc = O.render_entropy(osc, g, 2, 16, cam, RC, UC, contrib=True)
    rgb, dep, T, rcc = O.rasterize(osc, cam, RC, contrib=True)
    # entropy only (select_nbv without RGB), with contributor counts and depth
    r = api.render(ctx, scene, f, [cam], RC, UC, entropy=True, entropy_depth=True, contributors=True)
    assert np.array_equal(r["entropy_contributors"], cc)
    assert np.max(np.abs(r["entropy"] - H)) <= IMG_ABS
    assert np.max(np.abs(r["entropy_depth"] - edep)) <= 1e-4
    # RGB only
    r = api.render(ctx, scene, None, [cam], RC, UC, rgb=True, transmittance=True, contributors=True)
    assert np.array_equal(r["rgb_contributors"], rcc)
    assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS
    # correlation hook (needs the entropy-track depth inside the score)
    uc = UncertaintyConfig(correlation=1, correlation_lambda=2.0)
    res = api.select_nbv(ctx, scene, f, c["candidates"][:6], RC, uc)
    best, sc = O.select_nbv(osc, g, 2, 16, c["candidates"][:6], RC, uc, threads=8)
    assert res.best_index == best
    assert np.max(np.abs(res.scores - sc) / np.maximum(1.0, np.abs(sc))) <= SCORE_REL
    # tile 13 and alpha_clamp_max 1.0 run the exact kernels: fp64-level agreement
    for rc in (RasterConfig(tile_size=13), RasterConfig(alpha_clamp_max=1.0)):
        r = api.render(ctx, scene, f, [cam], rc, UC, entropy=True, contributors=True)
        He, _, _, cce = O.render_entropy(osc, g, 2, 16, cam, rc, UC, contrib=True)
        assert np.array_equal(r["entropy_contributors"], cce)
        assert np.max(np.abs(r["entropy"] - He)) <= 1e-10


def test_certified_sh_propagation(ctx):
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    rng = np.random.default_rng(11)
    var = rng.uniform(0.01, 0.2, size=(scene.num_particles, 3, 9)).astype(np.float32)
    ds = ctx.upload(scene)
    ds.set_coeff_variances(var, 2)
    f = api.construct_field(ctx, ds, c["train"][:4], VmfParams(1.0), 2, RC)
    g = f.download().gamma
    uc = UncertaintyConfig(variance_provider=1)
    cam = c["candidates"][0]
    r = api.render(ctx, ds, f, [cam], RC, uc, entropy=True, contributors=True, scores=True)
    O.set_coeff_variances(var.astype(np.float64), 2)
    try:
        H, _, _, cc = O.render_entropy(osc, g, 2, 4, cam, RC, uc, contrib=True)
    finally:
        O.set_coeff_variances(None, -1)
    assert np.array_equal(r["entropy_contributors"], cc)
    assert np.max(np.abs(r["entropy"] - H)) <= IMG_ABS


def test_certified_edge_cases(ctx):
    """1x1 camera, camera inside the cloud, nothing visible, empty scene."""
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    tiny = make_lookat((0, 0, 3), (0, 0, 0), (0, 1, 0), 1, 1)
    inside = make_lookat((0.1, 0.05, 0.0), (1, 0, 0), (0, 0, 1), 64, 48)
    away = make_lookat((0, 0, 10), (0, 0, 20), (0, 1, 0), 32, 32)
    for cam in (tiny, inside, away):
        r = api.render(ctx, scene, None, [cam], RC, UC, rgb=True, transmittance=True, contributors=True)
        rgb, _, T, cc = O.rasterize(osc, cam, RC, contrib=True)
        assert np.array_equal(r["rgb_contributors"], cc)
        assert np.max(np.abs(r["transmittance"] - T)) <= 1e-6
        assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS
    from paper_2605_30342_b200.model import Scene
    r = api.render(ctx, Scene.empty(), None, [synth.z_camera()], RC, UC, rgb=True, transmittance=True)
    assert np.all(r["rgb"] == 0) and np.all(r["transmittance"] == 1)


def test_certified_opacity_above_one(ctx):
    """The reference does not clamp opacities; the certified bound scales with the
    scene's largest opacity, so counts stay exact with o up to 3."""
    c = synth.config1(0)
    scene = c["scene"]
    boosted = scene.__class__(scene.positions, scene.rotations, scene.scales,
                              (scene.opacities * 3.0).astype(np.float32), scene.colors, scene.is_virtual,
                              scene.color_degree, scene.bounds_min, scene.bounds_max)
    osc = O.OracleScene(boosted)
    for cam in c["candidates"][:2]:
        r = api.render(ctx, boosted, None, [cam], RC, UC, rgb=True, contributors=True)
        rgb, _, _, cc = O.rasterize(osc, cam, RC, contrib=True)
        assert np.array_equal(r["rgb_contributors"], cc)
        assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS


@pytest.mark.parametrize("cutoff,amax", [(1e-2, 0.99), (1e-7, 0.99), (1e-4, 0.999), (1e-4, 0.5)])
def test_certified_raster_configs(ctx, cutoff, amax):
    """Other transmittance cutoffs and alpha clamps: the window is relative to the
    cutoff and the clamp bounds a/(1-a); counts stay exact."""
    c = synth.config1(0)
    scene = c["scene"]
    osc = O.OracleScene(scene)
    rc = RasterConfig(transmittance_cutoff=cutoff, alpha_clamp_max=amax)
    f = api.construct_field(ctx, scene, c["train"][:6], VmfParams(1.0), 2, rc)
    g = f.download().gamma
    cam = c["candidates"][3]
    r = api.render(ctx, scene, f, [cam], rc, UC, rgb=True, entropy=True, contributors=True)
    rgb, _, _, rcc = O.rasterize(osc, cam, rc, contrib=True)
    H, _, _, ecc = O.render_entropy(osc, g, 2, 6, cam, rc, UC, contrib=True)
    assert np.array_equal(r["rgb_contributors"], rcc)
    assert np.array_equal(r["entropy_contributors"], ecc)
    assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS
    assert np.max(np.abs(r["entropy"] - H)) <= IMG_ABS


def _fuzz_scene(seed: int, n: int):
    """Mixed populations: thin slabs, near-opaque splats (alpha at the clamp), faint
    large splats, degree-3 colours -- the regimes that stress the error bound."""
    rng = np.random.default_rng(seed)
    pos = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n), rng.uniform(2.0, 5.0, n)], 1)
    kind = rng.integers(0, 3, n)
    sc = np.exp(rng.normal(-3.5, 0.6, (n, 3)))
    sc[kind == 0, 2] = np.exp(rng.normal(-7.0, 0.3, int((kind == 0).sum())))  # slabs
    sc[kind == 2] *= 3.0                                                      # large, faint
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = np.where(kind == 1, rng.uniform(0.95, 1.0, n), rng.uniform(0.02, 0.9, n))
    op[kind == 2] *= 0.2
    col = rng.normal(0.0, 0.3, (n, 3, 16))
    col[:, :, 0] += 0.5 / 0.28209479177387814
    from paper_2605_30342_b200.model import Scene
    return Scene(pos.astype(np.float32), q.astype(np.float32), sc.astype(np.float32), op.astype(np.float32),
                 col.astype(np.float32), np.zeros(n, np.uint8), 3, np.array([-2.0, -2, 1]), np.array([2.0, 2, 7]))


@pytest.mark.parametrize("seed", range(6))
def test_certified_fuzz(ctx, seed):
    """Randomised scenes and cameras: contributor counts of both tracks exact,
    images within tolerance, against the oracle (given per-particle visibility)."""
    scene = _fuzz_scene(seed, 3000)
    osc = O.OracleScene(scene)
    rng = np.random.default_rng(100 + seed)
    vis = rng.uniform(0, 1, scene.num_particles)
    vis[rng.uniform(size=scene.num_particles) < 0.3] = 0.0
    vis[rng.uniform(size=scene.num_particles) < 0.2] = 1.0
    for k in range(2):
        eye = (rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5))
        cam = make_lookat(eye, (rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 3.5), (0, 1, 0), 96, 80)
        r = api.render(ctx, scene, None, [cam], RC, UC, rgb=True, entropy=True, contributors=True,
                       splat_visibility=vis)
        rgb, _, _, rcc = O.rasterize(osc, cam, RC, contrib=True)
        H, _, _ = O.render_entropy_core(osc, cam, RC, UC, vis)
        _, _, _, ecc = O.render_entropy_core(osc, cam, RC, UC, vis, contrib=True)
        assert np.array_equal(r["rgb_contributors"], rcc)
        assert np.array_equal(r["entropy_contributors"], ecc)
        assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS
        assert np.max(np.abs(r["entropy"] - H)) <= IMG_ABS


@pytest.mark.parametrize("degree", [0, 1, 2])
def test_certified_color_degrees(ctx, degree):
    """Colour degrees below 3: the tensor-core colour path zero-pads the 1/4/9
    coefficients of each channel to the GEMM's k = 16 (pre-split colour records)."""
    scene = synth._gaussian_cloud(7, 10_000, (-1, -1, -1), (1, 1, 1), -4.0, 0.5, color_degree=degree)
    osc = O.OracleScene(scene)
    for cam in synth.config1(0)["candidates"][:2]:
        r = api.render(ctx, scene, None, [cam], RC, UC, rgb=True, contributors=True)
        rgb, _, _, cc = O.rasterize(osc, cam, RC, contrib=True)
        assert np.array_equal(r["rgb_contributors"], cc)
        assert np.max(np.abs(r["rgb"] - rgb)) <= IMG_ABS


_FFMA_SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [sys.argv[1], sys.argv[1] + '/oracle']
import oracle as O
from paper_2605_30342_b200 import api, synth
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig
c = synth.config1(0)
osc = O.OracleScene(c['scene'])
with api.Context(0) as ctx:
    ctx.set_precision('certified')
    for cam in c['candidates'][:2]:
        r = api.render(ctx, c['scene'], None, [cam], RasterConfig(), UncertaintyConfig(), rgb=True,
                       contributors=True)
        rgb, _, _, cc = O.rasterize(osc, cam, RasterConfig(), contrib=True)
        assert np.array_equal(r['rgb_contributors'], cc)
        assert np.max(np.abs(r['rgb'] - rgb)) <= 2e-5, np.max(np.abs(r['rgb'] - rgb))
print('ok')
"""


def test_certified_ffma_colour_variant(tmp_path):
    """GAVIS_UA_COLOR=ffma (read once per process): the packed-FFMA colour path."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "ffma.py"
    script.write_text(_FFMA_SCRIPT)
    env = dict(os.environ, GAVIS_UA_COLOR="ffma")
    r = subprocess.run([sys.executable, str(script), root], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_certified_deterministic_and_batch_invariant(ctx, room):
    """Run to run and for any views-per-batch the certified outputs are bit-identical
    (per-view work is independent, the flagged-pixel redo is per pixel, the score
    fold has a fixed order) -- what makes sharded candidates agree at 1/2/4/8 GPUs."""
    scene = room["scene"]
    ds = ctx.upload(scene)
    f = api.construct_field(ctx, ds, room["train"], VmfParams(1.0), 2, RC)
    cams = room["candidates"]
    kw = dict(rgb=True, transmittance=True, entropy=True, invisible_mass=True, scores=True, contributors=True)
    a = api.render(ctx, ds, f, cams, RC, UC, **kw)
    b = api.render(ctx, ds, f, cams, RC, UC, **kw)
    ctx.set_batch(2)
    try:
        c = api.render(ctx, ds, f, cams, RC, UC, **kw)
        sel_b = api.select_nbv(ctx, ds, f, cams, RC, UC)
    finally:
        ctx.set_batch(0)
    sel_a = api.select_nbv(ctx, ds, f, cams, RC, UC)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
        assert np.array_equal(a[k], c[k]), k
    assert sel_a.best_index == sel_b.best_index
    assert np.array_equal(sel_a.scores, sel_b.scores)


def test_pair_budget_splits_batches(ctx, room):
    """A batch whose tile pairs exceed the pair budget is re-binned with fewer
    views (down to one); results are bit-identical to the unsplit run, for the
    field build and the render."""
    scene = room["scene"]
    ds = ctx.upload(scene)
    cams = room["candidates"]
    kw = dict(rgb=True, transmittance=True, entropy=True, invisible_mass=True, scores=True, contributors=True)
    f = api.construct_field(ctx, ds, room["train"], VmfParams(1.0), 2, RC)
    g = f.download().gamma
    a = api.render(ctx, ds, f, cams, RC, UC, **kw)
    _, ids, _ = api.debug_binning(ctx, ds, cams[0], RC)
    ctx.set_pair_budget(max(1, len(ids) + 1))  # about one view's pairs per batch
    try:
        f2 = api.construct_field(ctx, ds, room["train"], VmfParams(1.0), 2, RC)
        b = api.render(ctx, ds, f2, cams, RC, UC, **kw)
        sel = api.select_nbv(ctx, ds, f2, cams, RC, UC)
    finally:
        ctx.set_pair_budget(0)
    assert np.array_equal(f2.download().gamma, g)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert sel.best_index == api.select_nbv(ctx, ds, f, cams, RC, UC).best_index


def _scores_and_bounds(ctx, ctx_exact, scene, f, cams, uc=UC):
    cert = api.render(ctx, scene, f, cams, RC, uc, scores=True)["scores"]
    bounds = ctx.last_score_bounds()
    exact = api.render(ctx_exact, scene, f, cams, RC, uc, scores=True)["scores"]
    return cert, bounds, exact


@pytest.mark.parametrize("which", ["config1", "room", "fuzz"])
def test_certified_score_bounds_hold(ctx, ctx_exact, room, which):
    """The per-candidate score bound (kernels_ua_fast.cu, "score bound") is a
    rigorous bound on |certified - fp64 score|: it must hold on every candidate,
    and be tight enough to matter (well under the 1e-3 relative floor)."""
    if which == "config1":
        c = synth.config1(0)
    elif which == "room":
        c = room
    else:
        c = synth.config1(7)
        c["scene"].opacities[:] = np.minimum(c["scene"].opacities * 1.6, 0.999)  # near the clamp
    scene = c["scene"]
    f = api.construct_field(ctx_exact, scene, c["train"], VmfParams(1.0), 2, RC)
    cams = c["candidates"][:6]
    cert, bounds, exact = _scores_and_bounds(ctx, ctx_exact, scene, f, cams)
    assert bounds.shape == (len(cams),) and np.all(bounds > 0)
    assert np.all(np.abs(cert - exact) <= bounds), (np.abs(cert - exact), bounds)
    assert np.all(bounds <= 1e-3 * np.abs(exact))
    # the hook and sh_propagation carry no bound (their scoring calls run fp64)
    api.render(ctx, scene, f, cams[:1], RC, UncertaintyConfig(correlation=1, correlation_lambda=2.0),
               scores=True)
    assert ctx.last_score_bounds().size == 0


@pytest.mark.parametrize("mode", ["hook", "sh_propagation"])
def test_unbounded_modes_score_in_fp64(ctx, ctx_exact, mode):
    """select_nbv in certified mode with the correlation hook or sh_propagation --
    the modes whose certified scores have no rigorous bound -- runs the fp64 path
    (ScoringPrecision, host.h): scores bit-identical to the fp64 context's, no
    contender re-scoring, and the context stays in certified mode afterwards."""
    c = synth.config1(0)
    scene = c["scene"]
    uc = (UncertaintyConfig(correlation=1, correlation_lambda=2.0) if mode == "hook"
          else UncertaintyConfig(variance_provider=1))
    ds, de = ctx.upload(scene), ctx_exact.upload(scene)
    if mode == "sh_propagation":
        var = np.random.default_rng(3).uniform(0.01, 0.2, size=(scene.num_particles, 3, 9)).astype(np.float32)
        ds.set_coeff_variances(var, 2)
        de.set_coeff_variances(var, 2)
    f = api.construct_field(ctx_exact, de, c["train"], VmfParams(1.0), 2, RC)
    fc = api.upload_field(ctx, ds, f.download())
    cams = c["candidates"][:6]
    r0 = ctx.counters()
    a = api.select_nbv(ctx, ds, fc, cams, RC, uc)
    b = api.select_nbv(ctx_exact, de, f, cams, RC, uc)
    assert np.array_equal(a.scores, b.scores) and a.best_index == b.best_index
    assert ctx.counters() == r0  # no fp32 pixel redone, no candidate re-scored
    assert ctx.precision == "certified"


def test_certified_argmax_near_ties_around_zero(ctx, ctx_exact):
    """Scores near 0 (colour_sigma chosen so the fp64 score of the base view is
    ~0) with candidates a few 1e-9 rad apart: a purely relative window (1e-3
    |best|) would be empty; the bound-based window re-scores the near-ties in
    fp64 and the argmax is the fp64 one."""
    c = synth.config1(0)
    scene = c["scene"]
    f = api.construct_field(ctx_exact, scene, c["train"], VmfParams(1.0), 2, RC)
    base = c["candidates"][3]
    # score(hl) is affine in hl = 3 ln sigma (d score / d hl = sum of s): solve score = 0
    s1 = api.render(ctx_exact, scene, f, [base], RC, UncertaintyConfig(color_sigma=0.1), scores=True)["scores"][0]
    s2 = api.render(ctx_exact, scene, f, [base], RC, UncertaintyConfig(color_sigma=0.2), scores=True)["scores"][0]
    h1, h2 = 3 * np.log(0.1), 3 * np.log(0.2)
    hz = h1 - s1 * (h2 - h1) / (s2 - s1)
    uc = UncertaintyConfig(color_sigma=float(np.exp(hz / 3)))
    cams = []
    for k in range(6):
        eps = 2e-9 * (k - 2.5)
        cams.append(make_lookat(np.asarray(base.position) + np.array([eps, -eps, eps]),
                                np.asarray(base.position) + np.asarray(base.rotation)[:, 2], (0, 0, 1),
                                base.width, base.height, base.fov_h, base.fov_v))
    exact = api.select_nbv(ctx_exact, scene, f, cams, RC, uc)
    assert np.max(np.abs(exact.scores)) < 1e-3 * np.max(np.abs(s1)), "scores are not near zero"
    before = ctx.counters()[1]
    cert = api.select_nbv(ctx, scene, f, cams, RC, uc)
    assert cert.best_index == exact.best_index
    assert ctx.counters()[1] - before >= 2  # near-ties went to the fp64 re-scoring


def test_select_keeps_score_bounds(ctx):
    """select_nbv's fp64 re-scoring of its contenders does not clear the bounds of
    the certified scores it returns (gavis_ctx_last_score_bounds)."""
    c = synth.config1(0)
    f = api.construct_field(ctx, c["scene"], c["train"], VmfParams(1.0), 2, RC)
    cams = [c["candidates"][5]] * 3 + c["candidates"][:3]  # identical triple: contenders
    api.select_nbv(ctx, c["scene"], f, cams, RC, UC)
    b = ctx.last_score_bounds()
    assert b.shape == (len(cams),) and np.all(b > 0)


@pytest.mark.parametrize("case", ["negative_opacity", "visibility_outside_unit"])
def test_inputs_outside_the_bounds_assumptions(ctx, ctx_exact, case):
    """Inputs the reference does not exclude but the certified blend's bounds assume
    away -- negative opacities (alpha < 0) and caller-given visibilities outside
    [0, 1] (A alpha + B < 0) -- run the fp64 kernels with the lower alpha* clamp in
    both precisions (ua_render), and match the oracle: contributor counts
    bit-exact, images within 1e-9, scores and argmax equal."""
    c = synth.config1(0)
    scene = c["scene"]
    rng = np.random.default_rng(9)
    vis = rng.uniform(0.0, 1.0, scene.num_particles)
    if case == "negative_opacity":
        flip = rng.uniform(size=scene.num_particles) < 0.05
        scene.opacities[flip] = -0.3 * scene.opacities[flip]
    else:
        out = rng.uniform(size=scene.num_particles) < 0.1
        vis[out] = rng.choice([-0.4, 1.6], int(out.sum()))
    osc = O.OracleScene(scene)
    cam = c["candidates"][0]
    H, w0, _, cc = O.render_entropy_core(osc, cam, RC, UC, vis, contrib=True)
    rgb, _, T, rc_cc = O.rasterize(osc, cam, RC, contrib=True)
    for cx in (ctx, ctx_exact):
        r0 = cx.counters()
        r = api.render(cx, scene, None, [cam], RC, UC, rgb=True, entropy=True, invisible_mass=True,
                       contributors=True, splat_visibility=vis)
        assert cx.counters() == r0  # no certified pixel, no re-score: the fp64 kernels ran
        assert np.array_equal(r["entropy_contributors"], cc) and np.array_equal(r["rgb_contributors"], rc_cc)
        assert np.max(np.abs(r["entropy"] - H)) <= 1e-9
        assert np.max(np.abs(r["invisible_mass"] - w0)) <= 1e-9
        assert np.max(np.abs(r["rgb"] - rgb)) <= 1e-5
    if case == "negative_opacity":  # select_nbv with a field: fp64 in both precisions
        de, dc = ctx_exact.upload(scene), ctx.upload(scene)
        f = api.construct_field(ctx_exact, de, c["train"][:4], VmfParams(1.0), 2, RC)
        fc = api.upload_field(ctx, dc, f.download())
        r0 = ctx.counters()
        a = api.select_nbv(ctx, dc, fc, c["candidates"][:4], RC, UC)
        assert ctx.counters() == r0
        b = api.select_nbv(ctx_exact, de, f, c["candidates"][:4], RC, UC)
        best, sc = O.select_nbv(osc, f.download().gamma, 2, 4, c["candidates"][:4], RC, UC, threads=8)
        assert a.best_index == b.best_index == best
        assert np.max(np.abs(b.scores - sc) / np.abs(sc)) <= 1e-9
