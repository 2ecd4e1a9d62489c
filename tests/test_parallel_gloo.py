"""Multi-process (world_size 2, gloo, CPU) coverage of the sharding logic in
paper_2605_30342_b200.parallel. The per-shard compute is the CPU oracle here
(test infrastructure); on GPUs the same host logic drives the C ABI and NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_30342_b200 import parallel, synth
from paper_2605_30342_b200.model import RasterConfig, UncertaintyConfig, make_lookat

RC = RasterConfig()
UC = UncertaintyConfig()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _scene_and_views():
    sc = synth.random_scene(0xF00D, 60)
    views = [make_lookat((0.4 * k - 0.8, 0.3, 0.0), (0, 0, 4), (0, 1, 0), 48, 40) for k in range(5)]
    cands = [make_lookat((0.5 * np.cos(k), 0.5 * np.sin(k), 0.2), (0, 0, 4), (0, 1, 0), 48, 40)
             for k in range(7)]
    cands.append(cands[2])  # a tie across shards: the lowest index must win
    return sc, views, cands


def _worker(rank, world, port, out_dir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "oracle"))
    import oracle as O
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc, views, cands = _scene_and_views()
    osc = O.OracleScene(sc)

    def partial(lo, hi):
        return O.construct_field(osc, views[lo:hi], 1.0, 2, RC) if hi > lo else np.zeros((sc.num_particles, 9))

    def allreduce(field):
        t = torch.from_numpy(field)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    gamma = parallel.construct_field_sharded(partial, len(views), rank, world, allreduce)

    def score_block(lo, hi):
        return O.select_nbv(osc, gamma, 2, len(views), cands[lo:hi], RC, UC)[1]

    best, scores = parallel.select_nbv_sharded(score_block, len(cands), rank, world, dist)

    # certified argmax across shards: an fp32-like score block whose error pushes the
    # cross-shard duplicate (index 7, rank 1) above its twin (index 2, rank 0); the
    # contenders are re-scored exactly on their owning ranks and the tie goes back to 2
    exact = O.select_nbv(osc, gamma, 2, len(views), cands, RC, UC)[1]

    def approx_block(lo, hi):
        out = exact[lo:hi].copy()
        for i in range(lo, hi):
            out[i - lo] *= 1.0 + (1e-9 if i == 7 else -1e-9 * (i % 3))
        return out

    calls = []

    def rescore(idx):
        calls.append(list(idx))
        return exact[idx]

    cbest, cscores = parallel.select_nbv_sharded(approx_block, len(cands), rank, world, dist, rescore=rescore)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), gamma=gamma, best=best, scores=scores,
             cbest=cbest, cscores=cscores, ncalls=len(calls))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_sharded_field_and_nbv_match_single_process(tmp_path):
    import oracle as O
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    sc, views, cands = _scene_and_views()
    osc = O.OracleScene(sc)
    g_ref = O.construct_field(osc, views, 1.0, 2, RC)
    best_ref, scores_ref = O.select_nbv(osc, g_ref, 2, len(views), cands, RC, UC)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    # both ranks hold the identical all-reduced field
    assert np.array_equal(r0["gamma"], r1["gamma"])
    scale = np.maximum(np.abs(g_ref).max(axis=1, keepdims=True), 1e-300)
    assert float((np.abs(r0["gamma"] - g_ref) / scale).max()) <= 1e-12
    # scores gathered in candidate order, argmax identical, tie resolved to the lowest index
    assert np.array_equal(r0["scores"], r1["scores"])
    assert int(r0["best"]) == int(r1["best"]) == best_ref
    assert np.max(np.abs(r0["scores"] - scores_ref) / np.maximum(1.0, np.abs(scores_ref))) <= 1e-12
    assert r0["scores"][2] == r0["scores"][7]
    # certified sharded argmax equals the exact one, identical on both ranks
    assert int(r0["cbest"]) == int(r1["cbest"]) == best_ref
    assert np.array_equal(r0["cscores"], r1["cscores"])


def test_certified_contenders_rescored_across_shards():
    """Host logic without processes: a perturbation that would flip the argmax
    across a shard boundary is undone by re-scoring the contenders."""
    exact = np.array([1.0, 5.0, 3.0, 5.0, 2.0])
    approx = exact.copy()
    approx[3] *= 1 + 1e-8  # fp32 error favours the later duplicate
    assert parallel.first_max(approx) == 3
    best, sc = parallel.select_nbv_sharded(lambda lo, hi: approx[lo:hi], len(exact), 0, 1, None,
                                           rescore=lambda idx: exact[idx])
    assert best == 1 and sc[3] == exact[3]
    assert parallel.contenders(approx) == [1, 3]


def test_shard_range_partition():
    for n in (0, 1, 7, 100, 1024):
        for world in (1, 2, 3, 8):
            parts = [parallel.shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_first_max_rule():
    assert parallel.first_max([1.0, 3.0, 3.0, 2.0]) == 1
    assert parallel.first_max([5.0]) == 0
    assert parallel.first_max([2.0, 2.0, 2.0]) == 0


def test_contenders_window_bounds_and_floor():
    """The certified argmax window (ua_host.cu certified_contenders): per-candidate
    error bounds widen it; near score 0 the relative part vanishes and the bound /
    absolute floor keep the near-ties."""
    s = np.array([1e-12, -1e-12, 3e-12, -5.0])
    assert parallel.contenders(s) == [0, 1, 2]               # absolute floor 1e-9
    assert parallel.contenders(s, bounds=np.full(4, 2.6)) == [0, 1, 2, 3]
    big = np.array([100.0, 99.95, 99.0])
    assert parallel.contenders(big) == [0, 1]                  # 1e-3 relative
    assert parallel.contenders(big, bounds=np.array([0.6, 0.6, 0.6])) == [0, 1, 2]


def test_sharded_field_records_trajectory_length():
    """every rank's field must carry num_views = |P| after the
    all-reduce (query_visibility uses it as the exponent), not its block size."""
    class F:
        num_views = 0

    for rank in range(3):
        fld = parallel.construct_field_sharded(lambda lo, hi: F(), 10, rank, 3, lambda f: None,
                                               lambda f, n: setattr(f, "num_views", n))
        assert fld.num_views == 10
