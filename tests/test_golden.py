"""Committed golden vectors (tests/golden/config1_small.npz, made by
tests/golden/make_golden.py from the CPU oracle on seeded config-1 inputs):
the oracle must keep reproducing them exactly (CPU), and the device path --
exact and certified -- must match them within the north_star tolerances with
bit-exact contributor counts (GPU)."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import make_golden as G  # noqa: E402

from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams  # noqa: E402

GOLD = dict(np.load(os.path.join(HERE, "golden", "config1_small.npz")))


def test_oracle_reproduces_golden():
    got = G.compute()
    assert set(got) == set(GOLD)
    for k, v in GOLD.items():
        assert np.array_equal(got[k], v), k


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["exact", "certified"])
def test_device_matches_golden(precision):
    from paper_2605_30342_b200 import api
    scene, train, cam = G.inputs()
    rc, uc = RasterConfig(), UncertaintyConfig()
    with api.Context(0) as ctx:
        ctx.set_precision(precision)
        f = api.construct_field(ctx, scene, train, VmfParams(1.0), 2, rc)
        g = f.download().gamma[: G.GAMMA_ROWS]
        r = api.render(ctx, scene, f, [cam], rc, uc, rgb=True, transmittance=True, entropy=True,
                       invisible_mass=True, scores=True, contributors=True)
    scale = np.maximum(GOLD["gamma_rowmax"], 1e-300)[:, None]
    assert np.max(np.abs(g - GOLD["gamma_rows"]) / scale) <= 1e-5
    assert np.array_equal(r["rgb_contributors"], GOLD["rgb_contributors"].astype(np.int32))
    assert np.array_equal(r["entropy_contributors"], GOLD["entropy_contributors"].astype(np.int32))
    assert np.max(np.abs(r["rgb"] - GOLD["rgb"])) <= 1e-4
    assert np.max(np.abs(r["transmittance"] - GOLD["transmittance"])) <= 1e-6
    assert np.max(np.abs(r["entropy"] - GOLD["entropy"])) <= 1e-4
    assert np.max(np.abs(r["invisible_mass"] - GOLD["invisible_mass"])) <= 1e-5
    assert abs(r["scores"][0] - GOLD["score"][0]) <= 1e-6 * abs(GOLD["score"][0])
