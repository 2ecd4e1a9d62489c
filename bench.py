#!/usr/bin/env python
"""Benchmark: UA-render candidate views/s @800^2 (BASELINE.json metric), config 3.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 3]

A step scores one block of candidate views per GPU (select_nbv: fused RGB +
uncertainty render, image score, argmax) on the config-3 scene (1M Gaussians,
two-room indoor, 800x800). Per-GPU work is fixed (weak scaling): rank r scores
its own block of --per-gpu candidates. The VF construction (150 training views,
sharded over ranks + NCCL all-reduce) is timed separately as vf_build_ms.
Inputs (scene 240 MB + field 72 MB) exceed the 126 MB L2, so no flush is needed.

--impl reference times the CPU oracle (the reference's algorithm restated in C,
the reference itself does not build here) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "UA-render candidate views/s @800²"
UNIT = "candidate views/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--per-gpu", type=int, default=1024, help="candidates per GPU per step")
    p.add_argument("--particles", type=int, default=0, help="override Gaussian count (testing)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=0, help="candidates in the CPU sample")
    p.add_argument("--no-extra-vf", action="store_true", help="skip the config-2/4 VF-build timings")
    p.add_argument("--batch", type=int, default=0, help="views per launch batch (0 = library default)")
    p.add_argument("--sweep5", action="store_true",
                   help="config-5 active-mapping sweep: 20 incremental rounds x 512..4096 candidates at 400^2")
    p.add_argument("--precision", default="certified", choices=["certified", "exact"],
                   help="UA blend arithmetic (certified fp32 + fp64 redo, or fp64 throughout)")
    return p.parse_args()


def dist_init(gpus: int):
    """One process per GPU (torchrun env). GAVIS_DIST_BACKEND=gloo runs the same
    host logic over gloo (code-path smoke test with fewer GPUs than ranks: ranks
    then share devices round-robin; the collectives are host-side, no kernel of
    one rank waits on another)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as d
        backend = os.environ.get("GAVIS_DIST_BACKEND", "nccl")
        if backend != "nccl":
            local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            d.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            d.init_process_group(backend)
        dist = d
    return rank, local, world, dist


def make_config(cfg: int, world: int, per_gpu: int, particles: int):
    from paper_2605_30342_b200 import synth
    kw = {}
    if particles:
        kw["n"] = particles
    if cfg == 3:
        c = synth.config3(0, n_train=200, n_candidates=per_gpu * world, **kw)
        c["train200"] = c["train"]
        c["train"] = c["train"][:150]
    elif cfg == 2:
        c = synth.config2(0, n_candidates=per_gpu * world, **kw)
    elif cfg == 1:
        c = synth.config1(0)
    elif cfg == 4:
        c = synth.config4(0, n_candidates=per_gpu * world, **kw)
    else:
        c = synth.config5(0, n_candidates=per_gpu * world)
    return c


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 3 + k and "Active" in r[3 + k] and "Not" not in r[3 + k]:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def _coll_device(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def max_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(ctx, dist):
    import torch
    ctx.synchronize()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()


def cpu_info():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


def oracle_rate(c, gamma, degree, num_views, n_cands, threads):
    """The reference's algorithm (CPU oracle) on `n_cands` candidates: rasterize (RGB)
    + render_entropy + image_entropy + argmax, parallel over candidates (planner.hpp:125-131)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig
    osc = O.OracleScene(c["scene"])
    cams = c["candidates"][:n_cands]
    t0 = time.perf_counter()
    O.select_nbv(osc, gamma, degree, num_views, cams, RasterConfig(), UncertaintyConfig(), threads=threads,
                 with_rgb=True)
    dt = time.perf_counter() - t0
    return n_cands / dt, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2605_30342_b200.model import RasterConfig
    c = make_config(args.config, 1, max(8, args.cpu_sample or 8), args.particles)
    model, cores = cpu_info()
    # field for the oracle's render: the oracle's own construct_field over a view sample
    # would take minutes at 1M particles; the candidate-render cost does not depend on
    # the field's values, so build it from 2 training views.
    gamma = O.construct_field(O.OracleScene(c["scene"]), c["train"][:2], 1.0, c["degree"], RasterConfig(),
                              threads=cores)
    n = args.cpu_sample or max(cores, 8)
    rates = []
    for _ in range(args.warmup):
        oracle_rate(c, gamma, c["degree"], len(c["train"]), min(n, cores), cores)
    for _ in range(args.steps):
        r, dt = oracle_rate(c, gamma, c["degree"], len(c["train"]), n, cores)
        rates.append(r)
    value = float(np.mean(rates))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * n / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"config{args.config}", "candidates_per_step": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{n} candidates/step of config {args.config} at 800x800, "
                                       f"oracle select_nbv + rasterize on {cores} threads ({model})"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    from paper_2605_30342_b200 import api, parallel
    from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, VmfParams
    rank, local, world, dist = dist_init(args.gpus)
    torch.cuda.set_device(local)
    rc, uc = RasterConfig(), UncertaintyConfig()
    c = make_config(args.config, world, args.per_gpu, args.particles)
    scene = c["scene"]
    ctx = api.Context(local)
    ctx.set_precision(args.precision)
    if args.batch:
        ctx.set_batch(args.batch)
    ds = ctx.upload(scene)
    vmf = VmfParams(1.0)
    degree = c["degree"]
    train = c["train"]

    # ---------------- VF CONST: sharded views + NCCL all-reduce --------------
    def build_field(views, dscene=None, deg=None):
        dscene = dscene or ds
        deg = degree if deg is None else deg

        def partial(lo, hi):
            f = api.empty_field(ctx, dscene, vmf, deg)
            if hi > lo:
                api.accumulate_views(ctx, f, dscene, views[lo:hi], rc)
            return f
        f = parallel.construct_field_sharded(partial, len(views), rank, world,
                                             lambda fld: parallel.allreduce_device_field(fld, dist))
        f.set_num_views(len(views))
        return f

    field = build_field(train)  # warm-up + the field used for scoring
    barrier(ctx, dist)
    vf_times = []
    for _ in range(2):
        barrier(ctx, dist)
        t0 = time.perf_counter()
        tmp = build_field(train)
        barrier(ctx, dist)
        vf_times.append((time.perf_counter() - t0) * 1000.0)
        tmp.close()
    vf_ms = max_over_ranks(min(vf_times), dist)
    vf200_ms = None
    if "train200" in c:
        barrier(ctx, dist)
        t0 = time.perf_counter()
        tmp = build_field(c["train200"])
        barrier(ctx, dist)
        vf200_ms = max_over_ranks((time.perf_counter() - t0) * 1000.0, dist)
        tmp.close()

    # ---------------- UA render: candidate block of this rank ----------------
    lo, hi = parallel.shard_range(len(c["candidates"]), rank, world)
    cands = c["candidates"][lo:hi]

    def step():
        if world == 1:
            return api.select_nbv(ctx, ds, field, cands, rc, uc, with_rgb=True)
        # global argmax: scores all-gathered, contenders re-scored in fp64 on their ranks
        return api.select_nbv_sharded(ctx, ds, field, c["candidates"], rank, world, dist, rc, uc,
                                      with_rgb=True)

    for _ in range(args.warmup):
        res = step()
    ctx.set_profiling(True)
    KERNELS = ("ua_blend", "ua_redo", "preprocess", "sort", "depth_order", "scan",
               "emit_keys", "ranges", "score")
    for k in KERNELS:
        ctx.kernel_time(k, reset=True)
    redo0, resc0 = ctx.counters()
    barrier(ctx, dist)
    clocks = ClockSampler(local)
    clocks.start()
    l0 = ctx.launch_count()
    ctx.timer_start()
    for _ in range(args.steps):
        res = step()
    ms = ctx.timer_stop()
    launches = ctx.launch_count() - l0
    barrier(ctx, dist)
    clk = clocks.stop()
    ktimes = {k: ctx.kernel_time(k) for k in KERNELS}
    redo1, resc1 = ctx.counters()
    certified = {"redo_pixels_per_view": (redo1 - redo0) / float(len(cands) * args.steps),
                 "redo_fraction": (redo1 - redo0) / float(len(cands) * args.steps * cands[0].width * cands[0].height),
                 "rescored_candidates_per_step": (resc1 - resc0) / float(args.steps)}
    ctx.set_profiling(False)
    ms_max = max_over_ranks(ms, dist)
    total_cands = sum_over_ranks(float(len(cands) * args.steps), dist)
    value = total_cands / (ms_max / 1000.0)

    # parity gate of this run: certified scores/argmax against the exact fp64 path on
    # the first 8 candidates, contributor counts of one view (tests hold the oracle)
    gate_cams = cands[: min(8, len(cands))]
    cert = api.render(ctx, ds, field, gate_cams[:1], rc, uc, entropy=True, rgb=True, contributors=True)
    cert_scores = api.score_views(ctx, ds, field, gate_cams, rc, uc, with_rgb=True)
    ctx.set_precision("exact")
    exact = api.render(ctx, ds, field, gate_cams[:1], rc, uc, entropy=True, rgb=True, contributors=True)
    exact_scores = api.score_views(ctx, ds, field, gate_cams, rc, uc, with_rgb=True)
    ctx.set_precision(args.precision)
    # covered (pixel, list entry) pairs composited per view (SURVEY 8d secondary metric):
    # the per-pixel contributor counts of both tracks, averaged over the gate views
    cov_rgb = float(np.sum(exact["rgb_contributors"]))
    cov_ent = float(np.sum(exact["entropy_contributors"]))
    parity_gate = {
        "candidates": len(gate_cams),
        "scores_max_rel": float(np.max(np.abs(cert_scores - exact_scores) / np.abs(exact_scores))),
        "argmax_equal": bool(parallel.first_max(cert_scores) == parallel.first_max(exact_scores)),
        "contributors_equal": bool(np.array_equal(cert["rgb_contributors"], exact["rgb_contributors"]) and
                                   np.array_equal(cert["entropy_contributors"], exact["entropy_contributors"])),
        "images_max_abs": float(max(np.max(np.abs(cert["rgb"] - exact["rgb"])),
                                    np.max(np.abs(cert["entropy"] - exact["entropy"])))),
        "reference": "exact fp64 device path (pinned to the CPU oracle by tests/test_gpu_parity.py)"}

    # secondary: the reference planner's own select_nbv work (entropy + score, no RGB)
    barrier(ctx, dist)
    ctx.timer_start()
    api.select_nbv(ctx, ds, field, cands, rc, uc, with_rgb=False)
    ms_sel = max_over_ranks(ctx.timer_stop(), dist)
    select_only = sum_over_ranks(float(len(cands)), dist) / (ms_sel / 1000.0)

    # algorithmic bytes of the dominant kernel (ua_blend): per view 24 B per tile pair
    # (8 B key + 4 B id written once, read once) + 16 B per pixel (RGB + entropy, fp32)
    keys_per_view = []
    for cam in cands[: min(8, len(cands))]:
        k, _, _ = api.debug_binning(ctx, ds, cam, rc)
        keys_per_view.append(len(k))
    K_avg = float(np.mean(keys_per_view))
    P = cands[0].width * cands[0].height
    blend_ms, blend_n = ktimes["ua_blend"]
    views_per_launch = len(cands) * args.steps / max(1, blend_n)
    bytes_per_launch = views_per_launch * (24.0 * K_avg + 16.0 * P)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_per_launch / (blend_ms / max(1, blend_n) / 1000.0) / 1e9 if blend_n else 0.0
    step_ms = ms / args.steps
    N = scene.num_particles
    nb_c = (scene.color_degree + 1) ** 2
    pipe_bytes = N * (45 + 8 * (degree + 1) ** 2 + 12 * nb_c) + len(cands) * (24.0 * K_avg + 16.0 * P)

    # ---------------- e2e through the public C-ABI with host buffers ---------
    e2e = None
    if not args.no_e2e:
        host_field = field.download()
        pinned = {}
        for name in ("positions", "rotations", "scales", "opacities", "colors"):
            a = getattr(scene, name)
            t = torch.empty(a.shape, dtype=torch.float32, pin_memory=True)
            t.numpy()[...] = a
            pinned[name] = t.numpy()
        from paper_2605_30342_b200.model import Scene
        host_scene = Scene(pinned["positions"], pinned["rotations"], pinned["scales"], pinned["opacities"],
                           pinned["colors"], scene.is_virtual, scene.color_degree, scene.bounds_min,
                           scene.bounds_max)
        gpin = torch.empty(host_field.gamma.shape, dtype=torch.float64, pin_memory=True).numpy()
        gpin[...] = host_field.gamma
        host_field.gamma = gpin
        h2d = sum(v.nbytes for v in pinned.values()) + scene.is_virtual.nbytes + gpin.nbytes + 128 * len(cands)
        d2h = 8 * len(cands) + 4

        def e2e_step():
            s2 = ctx.upload(host_scene)
            f2 = api.upload_field(ctx, s2, host_field)
            r = api.select_nbv(ctx, s2, f2, cands, rc, uc, with_rgb=True)
            f2.close()
            s2.close()
            return r

        e2e_step()
        barrier(ctx, dist)
        e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        barrier(ctx, dist)
        e_ms = max_over_ranks((time.perf_counter() - t0) * 1000.0, dist)
        e_total = sum_over_ranks(float(len(cands) * e_steps), dist)
        e2e = {"value": e_total / (e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h),
               "timing": "host wall clock around upload(scene)+upload(field)+select_nbv, synchronised"}

    # ---------------- VF-build ms on configs 2 and 4 (BASELINE metric) ------
    vf_other = {}
    # configs 2 and 4 (scene generation on every rank's host is slow at 3M
    # Gaussians): one GPU only; the config-3 VF build above is measured at every N
    if not args.no_extra_vf and world == 1:
        from paper_2605_30342_b200 import synth
        for cid, gen in ((2, lambda: synth.config2(0, n_candidates=256)),
                         (4, lambda: synth.config4(0, n_candidates=64))):
            cc = gen()
            dsc = ctx.upload(cc["scene"])
            fld = build_field(cc["train"], dsc, cc["degree"])  # warm-up
            fld.close()
            times = []
            for _ in range(2):
                barrier(ctx, dist)
                t0 = time.perf_counter()
                fld = build_field(cc["train"], dsc, cc["degree"])
                barrier(ctx, dist)
                times.append((time.perf_counter() - t0) * 1000.0)
                if _ == 0:
                    fld.close()
            # UA render + score of this config's candidates (per rank block, device time)
            clo, chi = parallel.shard_range(len(cc["candidates"]), rank, world)
            ccands = cc["candidates"][clo:chi]
            api.select_nbv(ctx, dsc, fld, ccands, rc, uc, with_rgb=True)  # warm-up (buffer sizes)
            barrier(ctx, dist)
            ctx.timer_start()
            api.select_nbv(ctx, dsc, fld, ccands, rc, uc, with_rgb=True)
            ua_ms = max_over_ranks(ctx.timer_stop(), dist)
            fld.close()
            cam = cc["train"][0]
            vf_other[f"config{cid}"] = {"vf_build_ms": max_over_ranks(min(times), dist),
                                        "ua_views_per_s": sum_over_ranks(float(len(ccands)), dist) / (ua_ms / 1000.0),
                                        "ua_candidates": len(cc["candidates"]),
                                        "ua_resolution": [cc["candidates"][0].width, cc["candidates"][0].height],
                                        "views": len(cc["train"]), "particles": cc["scene"].num_particles,
                                        "resolution": [cam.width, cam.height], "field_degree": cc["degree"]}
            dsc.close()
            del cc

    # ---------------- config 5: active-mapping iteration sweep (1 GPU) ---------
    sweep5 = None
    if args.sweep5 and world == 1:
        from paper_2605_30342_b200 import synth
        c5 = synth.config5(0, n_candidates=4096)
        ds5 = ctx.upload(c5["scene"])
        sweep5 = {"scene": "config2 (500k Gaussians)", "training_views": len(c5["train"]),
                  "candidate_resolution": [400, 400], "rounds": c5["rounds"], "per_count": {}}
        for count in (512, 1024, 2048, 4096):
            f5 = build_field(c5["train"], ds5, c5["degree"])
            api.nbv_loop(ctx, ds5, f5, c5["candidates"][:count], 1, rc, uc)  # warm-up round
            f5.close()
            f5 = build_field(c5["train"], ds5, c5["degree"])
            barrier(ctx, dist)
            ctx.timer_start()
            chosen, _, _ = api.nbv_loop(ctx, ds5, f5, c5["candidates"][:count], c5["rounds"], rc, uc)
            ms5 = ctx.timer_stop()
            sweep5["per_count"][str(count)] = {
                "ms_per_round": ms5 / c5["rounds"],
                "candidate_views_per_s": count * c5["rounds"] / (ms5 / 1000.0),
                "chosen_first_rounds": [int(x) for x in chosen[:5]]}
            f5.close()
        ds5.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        model, cores = cpu_info()
        n = args.cpu_sample or max(4, min(16, cores))
        gamma = field.download().gamma
        rate, dt = oracle_rate(c, gamma, degree, len(train), n, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{n} of the config-{args.config} candidates (800x800, full scene), oracle "
                         f"select_nbv + rasterize on {cores} threads, {dt:.1f} s ({model})"}

    # dram bytes per ua_blend launch from the committed ncu --set full capture
    # (profiles/ncu_ua_blend.json, same launch shape: 16 config-3 views, RGB+entropy)
    traffic, traffic_src, compute = None, None, None
    prof = os.path.join(ROOT, "profiles", "ncu_ua_blend.json")
    if os.path.exists(prof):
        with open(prof) as f:
            pj = json.load(f)
        traffic = pj["traffic_bytes_per_launch"] * views_per_launch / pj["views_per_launch"]
        traffic_src = f"{pj['command']} ({pj['views_per_launch']} views/launch)"
        compute = {"bound": pj.get("compute_bound", "issue/latency"),
                   "fp64_pipe_active_pct": pj["fp64_pipe_active_pct"],
                   "issue_slots_busy_pct": pj["issue_slots_busy_pct"], "source": "same ncu capture"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "certified" else "f64",
            "precision": args.precision if args.precision == "exact" else
            "certified (fp32 blend, fp64 q; fp64 redo of uncertified pixels; exact argmax)",
            "certified": certified if args.precision == "certified" else None,
            "data": "synthetic (seeded config generator; paper datasets not in the container)",
            "config": {"workload": f"config{args.config}", "particles": N, "resolution": [cands[0].width, cands[0].height],
                       "candidates_per_gpu_per_step": len(cands), "training_views": len(train),
                       "field_degree": degree, "color_degree": scene.color_degree,
                       "parallelism": f"candidates sharded over {world} GPU(s), VF views sharded + NCCL all-reduce",
                       "l2": "inputs (scene+field) exceed the 126 MB L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src, "compute": compute,
                         "kernel": "ua_blend", "bytes_per_launch": bytes_per_launch,
                         "avg_launch_ms": blend_ms / max(1, blend_n), "launches": blend_n,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"},
            "pipeline": {"bytes_per_step": pipe_bytes, "achieved_gbs": pipe_bytes / (step_ms / 1000.0) / 1e9,
                         "pairs_per_view": K_avg, "kernel_ms_per_step": {k: v[0] / args.steps for k, v in ktimes.items()}},
            "select_nbv_entropy_only_views_per_s": select_only,
            "vf_build_ms": vf_ms, "vf_build_views": len(train), "vf_build_200_views_ms": vf200_ms,
            "vf_build_other_configs": vf_other,
            "best_index_last_step": int(res.best_index) + (lo if world == 1 else 0),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
            "parity_gate": parity_gate,
            "covered_pairs": {"rgb_per_view": cov_rgb, "entropy_per_view": cov_ent,
                              "per_s": (cov_rgb + cov_ent) * value,
                              "note": "pixel-entry evaluations until each track terminates, view 0 of the step"},
            **({"config5_sweep": sweep5} if sweep5 else {}),
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
