"""bench.py's multi-GPU launcher (CPU): `--gpus N` outside torchrun re-launches
itself as N ranks (torch.distributed.run, 127.0.0.1); over gloo the ranks
rendezvous, run the max/sum-over-ranks plumbing and rank 0 reports n_gpus = N.
With the NCCL backend and fewer visible devices than N it must fail loudly."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=240)


def test_gpus2_relaunches_two_ranks_over_gloo():
    r = _run(["--gpus", "2", "--selftest-dist", "--per-gpu", "8"], {"GAVIS_DIST_BACKEND": "gloo"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = lines[0]
    assert d["n_gpus"] == 2 and d["backend"] == "gloo"
    assert d["max_rank_plus_1"] == 2.0 and d["candidates"] == 16.0


def test_gpus_more_than_visible_fails_loudly():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("enough devices visible")
    r = _run(["--gpus", "2"], {"GAVIS_DIST_BACKEND": "nccl"})
    assert r.returncode != 0
    assert "visible CUDA devices" in r.stderr
