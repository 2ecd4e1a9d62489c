"""Per-pixel contributor statistics of config-3 candidates (how much work the
reference semantics imply per view)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_30342_b200 import api, synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams  # noqa: E402

c = synth.config3(0, n_train=150, n_candidates=8)
rc, uc = RasterConfig(), UncertaintyConfig()
with api.Context(0) as ctx:
    ds = ctx.upload(c["scene"])
    f = api.construct_field(ctx, ds, c["train"], VmfParams(1.0), 2, rc)
    for cam in c["candidates"][:4]:
        r = api.render(ctx, ds, f, [cam], rc, uc, rgb=True, entropy=True, contributors=True, transmittance=True)
        k, _, rg = api.debug_binning(ctx, ds, cam, rc)
        lens = rg[:, 1] - rg[:, 0]
        nr, ne = r["rgb_contributors"], r["entropy_contributors"]
        print(f"pairs {len(k)} tile-list mean {lens.mean():.0f} max {lens.max()} | rgb contrib mean {nr.mean():.1f} "
              f"p50 {np.median(nr):.0f} p99 {np.percentile(nr, 99):.0f} | ent contrib mean {ne.mean():.1f} "
              f"| T<cutoff frac {np.mean(r['transmittance'] < 1e-4):.3f}")
