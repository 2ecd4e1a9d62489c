"""Small deterministic workloads for ncu captures (one GPU).

  python tools/profile_driver.py ua   # 1 field build (16 views) + 2 x 16-candidate renders
  python tools/profile_driver.py vf   # 2 x 16-view field builds
Config 3 scene (1M Gaussians, 800x800), seed 0. GAVIS_PROFILE_PRECISION=exact selects
the fp64 blend.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_30342_b200 import api, synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "ua"
    n = int(os.environ.get("GAVIS_PROFILE_PARTICLES", "1000000"))
    c = synth.config3(0, n=n, n_train=16, n_candidates=32)
    rc, uc = RasterConfig(), UncertaintyConfig()
    with api.Context(0) as ctx:
        ctx.set_precision(os.environ.get("GAVIS_PROFILE_PRECISION", "certified"))
        ds = ctx.upload(c["scene"])
        t0 = time.time()
        field = api.construct_field(ctx, ds, c["train"], VmfParams(1.0), 2, rc)
        if mode == "vf":
            field = api.construct_field(ctx, ds, c["train"], VmfParams(1.0), 2, rc)
        else:
            for k in range(2):
                api.select_nbv(ctx, ds, field, c["candidates"][16 * k:16 * (k + 1)], rc, uc, with_rgb=True)
        ctx.synchronize()
        print(f"{mode} done in {time.time() - t0:.3f}s")


if __name__ == "__main__":
    main()
