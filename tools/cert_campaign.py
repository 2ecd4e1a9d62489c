"""Certification campaign on the GPU: the certified fp32 blend against the exact
fp64 device path (itself pinned to the CPU oracle by tests/test_gpu_parity.py) over
many randomised scenes and cameras, at sizes the oracle cannot reach in a test.

Per case: contributor counts of both tracks must be bit-identical, RGB / entropy
within 1e-4 max-abs (north_star), scores within 1e-5 relative, and select_nbv's
argmax identical. Scenes mix the regimes that stress the error bound: thin slabs,
near-opaque splats (alpha at the clamp), opacities above 1, faint large splats,
dense clusters (deep pixels with many composited entries), random visibility
(including exactly 0 and 1). Writes one JSON line.

    python tools/cert_campaign.py [--cases 60] [--seconds 600]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2605_30342_b200 import api  # noqa: E402
from paper_2605_30342_b200.model import (RasterConfig, Scene, UncertaintyConfig,  # noqa: E402
                                         VmfParams, make_lookat)


def scene_for(rng, n, spread=1.0):
    kind = rng.integers(0, 5, n)
    pos = np.stack([rng.uniform(-1.5, 1.5, n) * spread, rng.uniform(-1.5, 1.5, n) * spread,
                    2.0 + rng.uniform(0.0, 4.0, n) * spread], 1)
    dense = kind == 4                                        # tight cluster: deep pixels
    pos[dense] = rng.normal([0.2, -0.1, 3.5], 0.25, (int(dense.sum()), 3))
    sc = np.exp(rng.normal(rng.uniform(-4.5, -3.0), 0.6, (n, 3)))
    sc[kind == 0, 2] = np.exp(rng.normal(-7.5, 0.4, int((kind == 0).sum())))   # slabs
    sc[kind == 2] *= 4.0                                                        # large, faint
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(0.02, 0.95, n)
    op[kind == 1] = rng.uniform(0.97, 1.0, int((kind == 1).sum()))              # alpha at the clamp
    op[kind == 2] *= 0.15
    if rng.uniform() < 0.3:                                                     # unclamped opacities
        boost = rng.uniform(size=n) < 0.2
        op[boost] *= rng.uniform(1.0, 3.0, int(boost.sum()))
    col = rng.normal(0.0, 0.3, (n, 3, 16))
    col[:, :, 0] += 0.5 / 0.28209479177387814
    return Scene(pos.astype(np.float32), q.astype(np.float32), sc.astype(np.float32), op.astype(np.float32),
                 col.astype(np.float32), np.zeros(n, np.uint8), 3, np.array([-2.0, -2, 1]), np.array([2.0, 2, 7]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=400)
    ap.add_argument("--seconds", type=float, default=600.0)
    ap.add_argument("--seed", type=int, default=2026)
    ap.add_argument("--large", action="store_true", help="3M splats, 1920x1080 cameras (config-4 scale)")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    cert = api.Context(0)
    cert.set_precision("certified")
    exact = api.Context(0)
    exact.set_precision("exact")
    t0 = time.time()
    stats = dict(cases=0, views=0, pixels=0, count_mismatch_pixels=0, argmax_mismatch=0,
                 max_rgb_abs=0.0, max_entropy_abs=0.0, max_score_rel=0.0, redo_pixels=0,
                 rescored=0, particles_max=0)
    kw = dict(rgb=True, entropy=True, scores=True, contributors=True)
    for case in range(args.cases):
        if time.time() - t0 > args.seconds:
            break
        n = 3_000_000 if args.large else int(rng.choice([20_000, 100_000, 400_000]))
        # --large: 3M splats spread over a 4x wider volume (config-4 density per view:
        # tens of millions of tile pairs per 1080p view, far below the 2^31 limit)
        scene = scene_for(rng, n, 4.0 if args.large else 1.0)
        vis = rng.uniform(0, 1, n)
        vis[rng.uniform(size=n) < 0.25] = 0.0
        vis[rng.uniform(size=n) < 0.15] = 1.0
        res = int(rng.choice([256, 512, 800]))
        w, h = (1920, 1080) if args.large else (res, res)
        cams = []
        for _ in range(8):
            eye = (rng.uniform(-0.6, 0.6), rng.uniform(-0.6, 0.6), rng.uniform(-0.8, 0.8))
            cams.append(make_lookat(eye, (rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4), 3.6), (0, 1, 0),
                                    w, h, rng.uniform(0.6, 1.6), rng.uniform(0.6, 1.6)))
        uc = UncertaintyConfig(beta=float(rng.uniform(0.2, 0.8)), prior_opacity=float(rng.uniform(0.05, 0.3)))
        rc = RasterConfig(transmittance_cutoff=float(rng.choice([1e-4, 1e-4, 1e-3, 1e-5])),
                          alpha_clamp_max=float(rng.choice([0.99, 0.99, 0.999, 0.9, 0.5])))
        dc, de = cert.upload(scene), exact.upload(scene)
        r0 = cert.counters()
        a = api.render(cert, dc, None, cams, rc, uc, splat_visibility=vis, **kw)
        b = api.render(exact, de, None, cams, rc, uc, splat_visibility=vis, **kw)
        for k in ("rgb_contributors", "entropy_contributors"):
            stats["count_mismatch_pixels"] += int(np.count_nonzero(a[k] != b[k]))
        stats["max_rgb_abs"] = max(stats["max_rgb_abs"], float(np.max(np.abs(a["rgb"] - b["rgb"]))))
        stats["max_entropy_abs"] = max(stats["max_entropy_abs"], float(np.max(np.abs(a["entropy"] - b["entropy"]))))
        stats["max_score_rel"] = max(stats["max_score_rel"], float(np.max(
            np.abs(a["scores"] - b["scores"]) / np.maximum(1.0, np.abs(b["scores"])))))
        # argmax through select_nbv with a field built from 4 of the cameras (exact path)
        fe = api.construct_field(exact, de, cams[:4], VmfParams(1.0), 2, rc)
        fc = api.upload_field(cert, dc, fe.download())
        sa = api.select_nbv(cert, dc, fc, cams, rc, uc)
        sb = api.select_nbv(exact, de, fe, cams, rc, uc)
        stats["argmax_mismatch"] += int(sa.best_index != sb.best_index)
        stats["max_score_rel"] = max(stats["max_score_rel"], float(np.max(
            np.abs(sa.scores - sb.scores) / np.maximum(1.0, np.abs(sb.scores)))))
        r1 = cert.counters()
        stats["redo_pixels"] += r1[0] - r0[0]
        stats["rescored"] += r1[1] - r0[1]
        stats["cases"] += 1
        stats["views"] += len(cams)
        stats["pixels"] += len(cams) * w * h
        stats["particles_max"] = max(stats["particles_max"], n)
    stats["seconds"] = round(time.time() - t0, 1)
    stats["ok"] = (stats["count_mismatch_pixels"] == 0 and stats["argmax_mismatch"] == 0 and
                   stats["max_rgb_abs"] <= 1e-4 and stats["max_entropy_abs"] <= 1e-4)
    cert.close()
    exact.close()
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
