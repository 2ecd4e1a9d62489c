"""Device-memory stability over repeated scene uploads, field builds, select_nbv
and renders on one context: free device memory must plateau after the first
iteration (buffers are reused, scenes / fields return to the pool).

    python tools/leak_check.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_30342_b200 import api, synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams  # noqa: E402


def free_gb() -> float:
    f, _ = torch.cuda.mem_get_info(0)
    return f / 1e9


c = synth.config3(0, n=300_000, n_train=20, n_candidates=96, res=400)
rc, uc = RasterConfig(), UncertaintyConfig()
with api.Context(0) as ctx:
    for it in range(12):
        ds = ctx.upload(c["scene"])
        f = api.construct_field(ctx, ds, c["train"], VmfParams(1.0), 2, rc)
        r = api.select_nbv(ctx, ds, f, c["candidates"], rc, uc, with_rgb=True)
        api.render(ctx, ds, f, c["candidates"][:4], rc, uc, rgb=True, entropy=True, contributors=True)
        f.close()
        ds.close()
        print(it, r.best_index, round(free_gb(), 3), flush=True)
