"""Density control (vfield.hpp:136-199): oracle pinned to the
reference KATs (test_vfield.cpp:285-430) and the device path against the oracle."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2605_30342_b200 import synth
from paper_2605_30342_b200.model import K_PI, K_Y00, ParameterError, RasterConfig, Scene, VmfParams, make_lookat

RC = RasterConfig()


def opaque(pos, scale, opacity):
    return dict(pos=pos, scale=scale, opacity=opacity, color_sh=[[0.62 / K_Y00]] * 3)


def split_wall(dtype=np.float64):
    parts = [opaque((0.5, (i + 0.5) / 5.0, (j + 0.5) / 5.0), 0.12, 0.95) for i in range(5) for j in range(5)]
    return Scene.from_particles(parts, 0, bounds=((0, 0, 0), (1, 1, 1)), dtype=dtype)


def probe_positions(seed, n, bmin, bmax):
    out = []
    for k in range(n):
        g = synth.SplitMix64(synth.derive_seed(seed, k))
        u = (g.next_double(), g.next_double(), g.next_double())
        out.append([bmin[d] + (bmax[d] - bmin[d]) * u[d] for d in range(3)])
    return np.array(out)


def test_virtual_particle_scale_closed_form():
    """test_vfield.cpp:285-292"""
    s = math.cbrt(3.0 * (1.0 + 0.5) / (4.0 * K_PI * 100.0))
    assert abs(s - 0.1529915870972935) <= 1e-12 * s


def test_oracle_density_control_keeps_occluded_prunes_seen():
    """test_vfield.cpp:294-365 (exact double probes)."""
    sc = split_wall()
    cam = make_lookat((0.1, 0.5, 0.5), (1, 0.5, 0.5))
    kept, unseen = O.density_control(sc, (0, 0, 0), (1, 1, 1), [cam], rho=500.0, seed=99, round_f32=False)
    assert len(kept) >= 50
    n_virtual = int(np.floor(500.0))
    sampled = probe_positions(99, n_virtual, (0, 0, 0), (1, 1, 1))
    keptmask = np.zeros(n_virtual, bool)
    keptmask[kept] = True
    assert np.all(np.diff(kept) > 0)  # retention preserves sampling order

    def front(p):
        dx = p[0] - 0.1
        return p[0] < 0.4 and dx > 0.05 and abs(p[1] - 0.5) < 0.8 * dx and abs(p[2] - 0.5) < 0.8 * dx

    def behind(p):
        return p[0] > 0.6 and abs(p[1] - 0.5) < 0.3 and abs(p[2] - 0.5) < 0.3

    f = [k for k in range(n_virtual) if front(sampled[k])]
    b = [k for k in range(n_virtual) if behind(sampled[k])]
    assert len(f) > 10 and len(b) > 10
    assert np.mean(~keptmask[f]) >= 0.95
    assert np.mean(keptmask[b]) >= 0.95


def test_oracle_density_control_determinism_and_eps_one():
    """test_vfield.cpp:367-399"""
    sc = synth.wall_scene(np.float64)
    cam = make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5))
    a, _ = O.density_control(sc, (0, 0, 0), (2, 1, 1), [cam], rho=40.0, seed=5, round_f32=False)
    b, _ = O.density_control(sc, (0, 0, 0), (2, 1, 1), [cam], rho=40.0, seed=5, round_f32=False)
    assert np.array_equal(a, b)
    allk, _ = O.density_control(sc, (0, 0, 0), (2, 1, 1), [cam], rho=40.0, seed=5, eps_v=1.0, round_f32=False)
    assert len(allk) == int(np.floor(40.0 * 2.0))


# ----------------------------------------------------------------- device
@pytest.fixture(scope="module")
def ctx():
    from paper_2605_30342_b200 import api
    c = api.Context(0)
    yield c
    c.close()


@pytest.mark.gpu
def test_device_density_control_matches_oracle(ctx):
    from paper_2605_30342_b200 import api
    sc = split_wall(np.float32)
    cams = [make_lookat((0.1, 0.5, 0.5), (1, 0.5, 0.5)), make_lookat((0.2, 0.2, 0.8), (1, 0.5, 0.5), (0, 0, 1), 96, 80)]
    cfg = api.DensityControlConfig(rho=500.0, seed=99)
    aug, kept = api.density_control(ctx, sc, cams, cfg, RC, bounds=((0, 0, 0), (1, 1, 1)))
    okept, _ = O.density_control(sc, (0, 0, 0), (1, 1, 1), cams, rho=500.0, seed=99, round_f32=True)
    assert np.array_equal(kept, okept)
    assert aug.n == sc.num_particles + len(kept)
    # the augmented scene feeds the field: probe rows stay zero (test_vfield.cpp:412-430)
    f = api.construct_field(ctx, aug, cams[:1], VmfParams(1.0), 2, RC)
    g = f.download().gamma
    assert np.all(g[sc.num_particles:] == 0.0)
    q = api.query_visibility(ctx, f, [sc.num_particles], [[1, 0, 0]])
    assert q[0] == 0.0


@pytest.mark.gpu
def test_device_density_control_edges(ctx):
    from paper_2605_30342_b200 import api
    sc = synth.wall_scene()
    cam = make_lookat((0.3, 0.5, 0.5), (1, 0.5, 0.5))
    cfg = api.DensityControlConfig(rho=40.0, seed=5, eps_v=1.0)
    aug, kept = api.density_control(ctx, sc, [cam], cfg, RC, bounds=((0, 0, 0), (2, 1, 1)))
    assert len(kept) == 80 and aug.n == 25 + 80
    with pytest.raises(ParameterError):
        api.density_control(ctx, sc, [cam], cfg, RC, bounds=((0, 0, 0), (1, 1, 0)))
    with pytest.raises(ParameterError):
        api.density_control(ctx, sc, [cam], api.DensityControlConfig(eps_v=0.0), RC, bounds=((0, 0, 0), (2, 1, 1)))
