"""Visible splats (>= 1 tile pair) and tile pairs per config-3 candidate view."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_30342_b200 import api, synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig  # noqa: E402

c = synth.config3(0, n_train=1, n_candidates=8)
with api.Context(0) as ctx:
    ds = ctx.upload(c["scene"])
    for cam in c["candidates"]:
        _, ids, _ = api.debug_binning(ctx, ds, cam, RasterConfig())
        print(f"visible {len(np.unique(ids))}  pairs {len(ids)}")
