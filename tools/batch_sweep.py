"""Views-per-batch sweep of select_nbv at config 3 (1024 candidates, 800^2), with
and without the RGB track: device time per call (library stream events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_30342_b200 import api, synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams  # noqa: E402

c = synth.config3(0, n_candidates=1024)
rc, uc = RasterConfig(), UncertaintyConfig()
with api.Context(0) as ctx:
    ds = ctx.upload(c["scene"])
    f = api.construct_field(ctx, ds, c["train"], VmfParams(1.0), 2, rc)
    for rgb in (False, True):
        for bv in (16, 24, 32, 48, 64):
            ctx.set_batch(bv)
            api.select_nbv(ctx, ds, f, c["candidates"], rc, uc, with_rgb=rgb)
            best = 1e30
            for _ in range(2):
                ctx.timer_start()
                api.select_nbv(ctx, ds, f, c["candidates"], rc, uc, with_rgb=rgb)
                best = min(best, ctx.timer_stop())
            print(f"rgb={rgb} batch={bv}: {best:.1f} ms  {1024 / best * 1000:.0f} views/s", flush=True)
