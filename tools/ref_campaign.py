"""Parity campaign on the GPU against the reference ITSELF (oracle/_ref: its
unmodified headers compiled against the Eigen-subset shim) over randomised
scenes, cameras and configurations -- test infrastructure only.

Per case (both chains independent end to end, each with its own field):
  * single_view_visibility of one training view (raster.hpp:237-290): v;
  * construct_field over 4 training views (vfield.hpp:68-92): gamma per row;
  * select_nbv over 4 candidates (planner.hpp:117-137), fp64 and certified
    device paths: scores and the argmax; the certified scores against their own
    rigorous per-candidate bound (constant provider, no hook);
  * one candidate's rasterize / render_entropy images (raster.hpp:175-231,
    uncertainty.hpp:124-260): RGB, transmittance, entropy, w0;
  * per-pixel contributor counts of both tracks against the C restatement
    (oracle/gavis_oracle.c, bit-identical to the reference; the reference has no
    count output).
Randomised: particle count, colour degree 0-3, resolution (odd sizes), tile size,
cutoff, alpha clamp, dilation, beta / prior opacity / colour sigma, the
correlation hook, field degree 0-4, kappa, (10 % of cases) negative opacities,
(20 %) cameras inside the cloud, (20 %) fields of view up to ~150 degrees, and
the near plane. Writes one JSON line.

    python tools/ref_campaign.py [--cases 200] [--seconds 600] [--seed 11]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tools")]
import oracle as O  # noqa: E402
import ref as R  # noqa: E402
from cert_campaign import scene_for  # noqa: E402
from paper_2605_30342_b200 import api  # noqa: E402
from paper_2605_30342_b200.model import (RasterConfig, Scene, UncertaintyConfig,  # noqa: E402
                                         VmfParams, make_lookat)

THREADS = max(1, len(os.sched_getaffinity(0)))


def with_degree(s: Scene, d: int) -> Scene:
    nb = (d + 1) ** 2
    return Scene(s.positions, s.rotations, s.scales, s.opacities, np.ascontiguousarray(s.colors[:, :, :nb]),
                 s.is_virtual, d, s.bounds_min, s.bounds_max)


def campaign(cases: int, seconds: float, seed: int, max_particles: int = 60_000) -> dict:
    """Run up to `cases` random cases (or until `seconds` elapse); returns the stats
    dict with its `ok` verdict (tests/test_ref_campaign.py runs a short one)."""
    rng = np.random.default_rng(seed)
    ctx = api.Context(0)
    t0 = time.time()
    st = dict(cases=0, candidates=0, pixels=0, count_mismatch_pixels=0, argmax_mismatch_exact=0,
              argmax_mismatch_certified=0, max_v_abs=0.0, max_gamma_rel=0.0, max_rgb_abs=0.0, max_trans_abs=0.0,
              max_entropy_abs=0.0, max_w0_abs=0.0, max_score_rel_exact=0.0, max_score_rel_certified=0.0,
              tile_sizes=[], color_degrees=[], field_degrees=[], hook_cases=0, bounded_candidates=0,
              bound_violations=0, max_error_over_bound=0.0, worst_certified_case=None,
              count_mismatch_pixels_certified=0, max_rgb_abs_certified=0.0, max_entropy_abs_certified=0.0,
              negative_opacity_cases=0, inside_cloud_cases=0, wide_fov_cases=0)
    for case in range(cases):
        if time.time() - t0 > seconds:
            break
        n = min(max_particles, int(rng.choice([5_000, 20_000, 60_000])))
        cd = int(rng.integers(0, 4))
        scene = with_degree(scene_for(rng, n), cd)
        negative = rng.uniform() < 0.1  # opacities the reference does not exclude: alpha < 0
        if negative:
            flip = rng.uniform(size=n) < 0.05
            scene.opacities[flip] = -0.3 * scene.opacities[flip]
        w, h = int(rng.integers(48, 300)), int(rng.integers(48, 300))
        cams = []
        inside = rng.uniform() < 0.2  # cameras inside the cloud: near-plane culls, clamped Jacobians
        wide = rng.uniform() < 0.2    # wide fields of view (up to ~150 degrees)
        for _ in range(8):
            eye = (rng.uniform(-0.6, 0.6), rng.uniform(-0.6, 0.6),
                   rng.uniform(2.5, 4.5) if inside else rng.uniform(-0.8, 0.8))
            fmax = 2.6 if wide else 1.6
            cam = make_lookat(eye, (rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4), eye[2] + 2.0 if inside else 3.6),
                              (0, 1, 0), w, h, rng.uniform(0.6, fmax), rng.uniform(0.6, fmax))
            cam.near = float(rng.choice([0.05, 0.05, 0.2, 1.0]))
            cams.append(cam)
        train, cands = cams[:4], cams[4:]
        rc = RasterConfig(tile_size=int(rng.choice([16, 16, 16, 8, 13, 32])),
                          transmittance_cutoff=float(rng.choice([1e-4, 1e-4, 1e-3, 1e-5])),
                          dilation=float(rng.choice([0.3, 0.3, 0.1, 0.0])),
                          alpha_clamp_max=float(rng.choice([0.99, 0.99, 0.999, 0.9, 0.5])))
        hook = rng.uniform() < 0.2
        uc = UncertaintyConfig(beta=float(rng.uniform(0.0, 1.0)), prior_opacity=float(rng.uniform(0.0, 0.4)),
                               color_sigma=float(rng.choice([0.1, 0.05, 0.3])),
                               correlation=1 if hook else 0, correlation_lambda=float(rng.uniform(0.5, 4.0)))
        L = int(rng.integers(0, 5))
        kappa = float(rng.uniform(0.5, 4.0))
        osc = O.OracleScene(scene)
        ds = ctx.upload(scene)

        # VF: one view's visibility, then the 4-view field
        ctx.set_precision("exact")
        v = api.single_view_visibility(ctx, ds, train[0], rc)
        rv = R.single_view_visibility(osc, train[0], rc, threads=THREADS)
        st["max_v_abs"] = max(st["max_v_abs"], float(np.max(np.abs(v - rv))))
        f = api.construct_field(ctx, ds, train, VmfParams(kappa), L, rc)
        g = f.download().gamma
        rg = R.construct_field(osc, train, kappa, L, rc, threads=THREADS)
        scale = np.maximum(np.abs(rg).max(axis=1, keepdims=True), 1e-300)
        st["max_gamma_rel"] = max(st["max_gamma_rel"], float((np.abs(g - rg) / scale).max()))

        # UA + argmax: the reference's chain on its own field, the device's on its own
        rbest, rscores = R.select_nbv(osc, rg, L, len(train), cands, rc, uc, threads=THREADS)
        for prec in ("exact", "certified"):
            ctx.set_precision(prec)
            nbv = api.select_nbv(ctx, ds, f, cands, rc, uc)
            rel = float(np.max(np.abs(nbv.scores - rscores) / np.maximum(np.abs(rscores), 1e-300)))
            st[f"argmax_mismatch_{prec}"] += int(nbv.best_index != rbest)
            if prec == "certified":
                # the certified scores' own rigorous bound (constant provider, no hook):
                # |certified - fp64| <= bound, and the fp64 path is ~1e-12 from the reference
                bd = ctx.last_score_bounds()
                if len(bd) == len(cands):
                    st["bounded_candidates"] += len(cands)
                    st["bound_violations"] += int(np.count_nonzero(
                        np.abs(nbv.scores - rscores) > bd + 1e-9 * np.abs(rscores)))
                    st["max_error_over_bound"] = max(st["max_error_over_bound"], float(np.max(
                        np.abs(nbv.scores - rscores) / np.maximum(bd, 1e-300))))
                if rel > st["max_score_rel_certified"]:
                    st["worst_certified_case"] = dict(
                        case=case, particles=n, width=w, height=h, tile=rc.tile_size,
                        cutoff=rc.transmittance_cutoff, alpha_clamp=rc.alpha_clamp_max, hook=bool(hook),
                        beta=uc.beta, prior_opacity=uc.prior_opacity, color_sigma=uc.color_sigma,
                        field_degree=L, scores_ref=[float(x) for x in rscores],
                        bounds=[float(x) for x in bd])
            st[f"max_score_rel_{prec}"] = max(st[f"max_score_rel_{prec}"], rel)
        ctx.set_precision("exact")

        # one candidate's images and contributor counts
        cam = cands[0]
        P = cam.width * cam.height
        out = api.render(ctx, ds, f, [cam], rc, uc, rgb=True, transmittance=True, entropy=True,
                         invisible_mass=True, contributors=True)
        rrgb, _, rT = R.rasterize(osc, cam, rc, threads=THREADS)
        rH, rw0, _ = R.render_entropy(osc, rg, L, len(train), cam, rc, uc, threads=THREADS)
        st["max_rgb_abs"] = max(st["max_rgb_abs"], float(np.max(np.abs(out["rgb"] - rrgb))))
        st["max_trans_abs"] = max(st["max_trans_abs"], float(np.max(np.abs(out["transmittance"][:P] - rT))))
        st["max_entropy_abs"] = max(st["max_entropy_abs"], float(np.max(np.abs(out["entropy"][:P] - rH))))
        st["max_w0_abs"] = max(st["max_w0_abs"], float(np.max(np.abs(out["invisible_mass"][:P] - rw0))))
        o_rgb = O.rasterize(osc, cam, rc, contrib=True)
        o_ent = O.render_entropy(osc, g, L, len(train), cam, rc, uc, contrib=True)
        st["count_mismatch_pixels"] += int(np.count_nonzero(out["rgb_contributors"][:P] != o_rgb[3]))
        st["count_mismatch_pixels"] += int(np.count_nonzero(out["entropy_contributors"][:P] != o_ent[3]))
        # the same candidate through the certified path
        ctx.set_precision("certified")
        oc = api.render(ctx, ds, f, [cam], rc, uc, rgb=True, entropy=True, contributors=True)
        ctx.set_precision("exact")
        st["count_mismatch_pixels_certified"] += int(np.count_nonzero(oc["rgb_contributors"][:P] != o_rgb[3]))
        st["count_mismatch_pixels_certified"] += int(np.count_nonzero(oc["entropy_contributors"][:P] != o_ent[3]))
        st["max_rgb_abs_certified"] = max(st["max_rgb_abs_certified"], float(np.max(np.abs(oc["rgb"] - rrgb))))
        st["max_entropy_abs_certified"] = max(st["max_entropy_abs_certified"],
                                              float(np.max(np.abs(oc["entropy"][:P] - rH))))

        f.close()
        st["cases"] += 1
        st["candidates"] += len(cands)
        st["pixels"] += len(cands) * P
        st["hook_cases"] += int(hook)
        st["negative_opacity_cases"] += int(negative)
        st["inside_cloud_cases"] += int(inside)
        st["wide_fov_cases"] += int(wide)
        for k, x in (("tile_sizes", rc.tile_size), ("color_degrees", cd), ("field_degrees", L)):
            if x not in st[k]:
                st[k].append(x)
    st["seconds"] = round(time.time() - t0, 1)
    st["threads"] = THREADS
    st["ok"] = (st["count_mismatch_pixels"] == 0 and st["argmax_mismatch_exact"] == 0 and
                st["argmax_mismatch_certified"] == 0 and st["max_gamma_rel"] <= 1e-5 and
                st["max_rgb_abs"] <= 1e-4 and st["max_entropy_abs"] <= 1e-4 and
                st["max_score_rel_exact"] <= 1e-6 and st["bound_violations"] == 0 and
                st["count_mismatch_pixels_certified"] == 0 and st["max_rgb_abs_certified"] <= 1e-4 and
                st["max_entropy_abs_certified"] <= 1e-4)
    ctx.close()
    return st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seconds", type=float, default=600.0)
    ap.add_argument("--seed", type=int, default=11)
    args = ap.parse_args()
    if not R.available():
        print(json.dumps({"ok": False, "skipped": "oracle/_ref not built"}))
        return
    st = campaign(args.cases, args.seconds, args.seed)
    st["command"] = " ".join(["python"] + sys.argv)
    print(json.dumps(st))


if __name__ == "__main__":
    main()
