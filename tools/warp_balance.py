"""Critical path of the fp64 blend's schedules, simulated on the CPU from the
oracle's projection and binning of config-3 candidates (test infrastructure:
oracle only). Per tile, warp w (an 8x4 patch) does work on every list entry that
meets its patch while one of its pixels is live (RGB track). Reports, summed
over tiles: the barrier schedule (batches of B entries, each as long as its
slowest warp), the decoupled schedule (each tile as long as its slowest warp's
total) and the perfectly balanced mean.

  python tools/warp_balance.py [n_candidates]
"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import oracle as O
from paper_2605_30342_b200 import synth
from paper_2605_30342_b200.model import RasterConfig

def simulate(scene, cam, rc, B=64):
    sp = O.project_scene(O.OracleScene(scene), cam, rc.dilation)
    off, ent = O.splat_binning(sp, cam.width, cam.height, rc.tile_size)
    mx = np.array([s.mean_x for s in sp]); my = np.array([s.mean_y for s in sp])
    ca = np.array([s.conic_a for s in sp]); cb = np.array([s.conic_b for s in sp])
    cc = np.array([s.conic_c for s in sp]); rr = np.array([s.radius for s in sp])
    op = np.array([s.opacity for s in sp])
    tx = (cam.width + 15) // 16
    tot_bar = tot_dec = tot_avg = 0
    for t in range(len(off) - 1):
        lst = ent[off[t]:off[t + 1]]
        if len(lst) == 0: continue
        x0, y0 = (t % tx) * 16, (t // tx) * 16
        L = len(lst)
        work = np.zeros((8, L), bool)
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
            live = (Tprev >= rc.transmittance_cutoff) & inside[None, :]
            work[w] = hit & (live.sum(axis=1) > 0)
        # barrier schedule: batches of B until every warp is done
        lastlive = np.max(np.nonzero(work.any(axis=0))[0]) + 1 if work.any() else 0
        nb = (lastlive + B - 1) // B
        for b in range(nb):
            tot_bar += work[:, b*B:(b+1)*B].sum(axis=1).max()
        tot_dec += work.sum(axis=1).max()
        tot_avg += work.sum() / 8.0
    return tot_bar, tot_dec, tot_avg

c = synth.config3(0, n_train=1, n_candidates=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
for cam in c["candidates"]:
    for B in (32, 64, 128):
        bar, dec, avg = simulate(c["scene"], cam, RasterConfig(), B)
        print(f"B={B}: barrier {bar:.0f}  decoupled {dec:.0f}  mean {avg:.0f}  bar/dec {bar/dec:.3f}  dec/mean {dec/avg:.3f}")
