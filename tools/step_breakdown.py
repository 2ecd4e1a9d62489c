"""Where the config-3 bench step's time goes beyond the blend kernel: device time
(library stream events) of select_nbv over 1024 candidates against plain renders
(no argmax re-scoring) of 32 / 1024 / 2048 candidates -- fixed cost per call vs
marginal cost per view -- and the per-kernel sums of one select_nbv."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_30342_b200 import api, synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams  # noqa: E402

c = synth.config3(0, n_candidates=2048)
rc, uc = RasterConfig(), UncertaintyConfig()
with api.Context(0) as ctx:
    ds = ctx.upload(c["scene"])
    f = api.construct_field(ctx, ds, c["train"], VmfParams(1.0), 2, rc)
    cands = c["candidates"]

    def timed(fn, reps=2):
        fn()
        best = 1e30
        for _ in range(reps):
            ctx.timer_start()
            fn()
            best = min(best, ctx.timer_stop())
        return best

    sel = timed(lambda: api.select_nbv(ctx, ds, f, cands[:1024], rc, uc, with_rgb=True))
    r32 = timed(lambda: api.render(ctx, ds, f, cands[:32], rc, uc, with_rgb=True, scores=True))
    r1k = timed(lambda: api.render(ctx, ds, f, cands[:1024], rc, uc, with_rgb=True, scores=True))
    r2k = timed(lambda: api.render(ctx, ds, f, cands[:2048], rc, uc, with_rgb=True, scores=True))
    print(f"select_nbv 1024 (with RGB): {sel:.1f} ms")
    print(f"render 32 / 1024 / 2048: {r32:.1f} / {r1k:.1f} / {r2k:.1f} ms;"
          f" marginal {(r2k - r1k) / 1024:.3f} ms/view; fixed ~{r1k - 1024 * (r2k - r1k) / 1024:.1f} ms")
    ctx.set_profiling(True)
    ks = ("ua_blend", "ua_redo", "preprocess", "sort", "depth_order", "scan",
          "emit_keys", "ranges", "score")
    for k in ks:
        ctx.kernel_time(k, reset=True)
    api.select_nbv(ctx, ds, f, cands[:1024], rc, uc, with_rgb=True)
    print({k: round(ctx.kernel_time(k)[0], 1) for k in ks})
    ctx.set_profiling(False)
    for k in ks:
        ctx.kernel_time(k, reset=True)
    bl = timed(lambda: api.render(ctx, ds, f, cands[:1024], rc, uc, with_rgb=True, scores=True))
    print(f"render 1024 without per-kernel events: {bl:.1f} ms")
