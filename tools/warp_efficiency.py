"""Lane efficiency of K7f's schedule (warp = 8x4 pixel patch walking the tile list,
pre-filtered to entries whose cover rectangle meets the patch, until all 32
pixels have terminated), simulated on the CPU from the oracle's projection and
binning for config-3 candidates, RGB track (test infrastructure: oracle only).

Reports, per view: useful lane-entries (pixel covered and not terminated) over
32 x warp-entries evaluated, and the share of warp-entries spent after the
warp's live pixel count fell to <= 4 / <= 8 (stragglers)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O  # noqa: E402
from paper_2605_30342_b200 import synth  # noqa: E402
from paper_2605_30342_b200.model import RasterConfig  # noqa: E402


def simulate(scene, cam, rc):
    sp = O.project_scene(O.OracleScene(scene), cam, rc.dilation)
    off, ent = O.splat_binning(sp, cam.width, cam.height, rc.tile_size)
    mx = np.array([s.mean_x for s in sp]); my = np.array([s.mean_y for s in sp])
    ca = np.array([s.conic_a for s in sp]); cb = np.array([s.conic_b for s in sp])
    cc = np.array([s.conic_c for s in sp]); rr = np.array([s.radius for s in sp])
    op = np.array([s.opacity for s in sp])
    tx = (cam.width + 15) // 16
    useful = evaluated = late4 = late8 = 0
    for t in range(len(off) - 1):
        lst = ent[off[t]:off[t + 1]]
        if len(lst) == 0:
            continue
        x0, y0 = (t % tx) * 16, (t // tx) * 16
        for w in range(8):
            bx, by = x0 + (w & 1) * 8, y0 + (w >> 1) * 4
            px = bx + (np.arange(32) & 7); py = by + (np.arange(32) >> 3)
            inside = (px < cam.width) & (py < cam.height)
            cx = px[None, :] + 0.5 - mx[lst][:, None]; cy = py[None, :] + 0.5 - my[lst][:, None]
            cov = (np.abs(cx) <= rr[lst][:, None]) & (np.abs(cy) <= rr[lst][:, None]) & inside[None, :]
            hit = cov.any(axis=1)
            q = ca[lst][:, None] * cx * cx + 2 * cb[lst][:, None] * cx * cy + cc[lst][:, None] * cy * cy
            al = np.minimum(op[lst][:, None] * np.exp(-0.5 * q), rc.alpha_clamp_max) * cov
            T = np.cumprod(1.0 - al, axis=0)
            Tprev = np.vstack([np.ones((1, 32)), T[:-1]])
            live = (Tprev >= rc.transmittance_cutoff) & inside[None, :]   # before compositing entry j
            nlive = live.sum(axis=1)
            rows = np.nonzero(hit & (nlive > 0))[0]
            evaluated += len(rows)
            useful += int((cov & live)[rows].sum())
            late4 += int((nlive[rows] <= 4).sum())
            late8 += int((nlive[rows] <= 8).sum())
    return useful / max(1, 32 * evaluated), late4 / max(1, evaluated), late8 / max(1, evaluated), evaluated


if __name__ == "__main__":
    c = synth.config3(0, n_train=1, n_candidates=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
    for cam in c["candidates"]:
        eff, l4, l8, ev = simulate(c["scene"], cam, RasterConfig())
        print(f"warp-entries {ev}  lane efficiency {eff:.3f}  after <=4 live {l4:.3f}  after <=8 live {l8:.3f}")
