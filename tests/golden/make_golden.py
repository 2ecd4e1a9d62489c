"""Regenerates tests/golden/config1_small.npz: CPU-oracle outputs (oracle/, pinned to
the reference's known-answer tests by tests/test_oracle_kats.py) on seeded config-1
inputs, so the GPU parity of the hot path can be checked against committed vectors
and oracle drift is caught on CPU (tests/test_golden.py).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]


def inputs():
    from paper_2605_30342_b200 import synth
    from paper_2605_30342_b200.model import make_lookat
    c = synth.config1(0)
    cand = c["candidates"][5]
    small = make_lookat(cand.position, (0.0, 0.0, 0.0), (0, 0, 1), 128, 128, cand.fov_h, cand.fov_v)
    return c["scene"], c["train"][:4], small


GAMMA_ROWS = 2000


def compute():
    import oracle as O
    from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig
    scene, train, cam = inputs()
    rc, uc = RasterConfig(), UncertaintyConfig()
    osc = O.OracleScene(scene)
    gamma = O.construct_field(osc, train, 1.0, 2, rc, threads=os.cpu_count() or 1)
    rgb, _, T, rcc = O.rasterize(osc, cam, rc, contrib=True)
    H, w0, _, ecc = O.render_entropy(osc, gamma, 2, len(train), cam, rc, uc, contrib=True)
    return dict(gamma_rows=gamma[:GAMMA_ROWS], gamma_rowmax=np.abs(gamma).max(axis=1)[:GAMMA_ROWS],
                rgb=rgb.astype(np.float32), transmittance=T.astype(np.float32),
                rgb_contributors=rcc.astype(np.int16), entropy=H.astype(np.float32),
                invisible_mass=w0.astype(np.float32), entropy_contributors=ecc.astype(np.int16),
                score=np.array([O.image_entropy(H)]))


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "config1_small.npz"), **compute())
    print("wrote", os.path.join(HERE, "config1_small.npz"))
