"""Multi-GPU decomposition of the two hot paths.

One process per GPU (torch.distributed for the plumbing):
  * UA render + argmax: candidates are independent (planner.hpp:125-131), so each
    rank scores a contiguous block with no data-path communication; the V fp64
    scores are gathered once and reduced with the reference's first-maximum rule
    (planner.hpp:132-136). Per-candidate scores do not depend on the rank count.
  * VF CONST: gamma is a linear sum over views (vfield.hpp:53-60; test_vfield.cpp:
    104-131), so each rank accumulates a contiguous block of training views into a
    partial field and one all-reduce(sum, fp64) over NCCL/NVLink completes it;
    num_views is then the trajectory length.

The compute callables are injected so the same host logic runs over the CUDA
library in production and over gloo on CPU in the tests.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Static block partition [n*r/w, n*(r+1)/w) -- parallel.hpp:50-51's rule."""
    return (n * rank) // world, (n * (rank + 1)) // world


def first_max(scores: Sequence[float]) -> int:
    """planner.hpp:132-136: strict '>' keeps the lowest index among ties."""
    best = 0
    for i in range(1, len(scores)):
        if scores[i] > scores[best]:
            best = i
    return best


def gather_scores(local: np.ndarray, n_total: int, rank: int, world: int, dist=None) -> np.ndarray:
    """All-gather variable-sized contiguous score blocks into rank order."""
    if world == 1 or dist is None:
        return np.asarray(local, np.float64)
    import torch
    lo, hi = shard_range(n_total, rank, world)
    width = max(shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0] for r in range(world))
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(width, dtype=torch.float64, device=dev)
    buf[: hi - lo] = torch.as_tensor(np.asarray(local, np.float64), device=dev)
    parts = [torch.zeros(width, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = []
    for r in range(world):
        a, b = shard_range(n_total, r, world)
        out.append(parts[r][: b - a].cpu().numpy())
    return np.concatenate(out) if out else np.zeros(0)


CERT_SCORE_REL = 1e-3  # same window as the library's select (ua_host.cu kCertScoreRel)
CERT_SCORE_ABS = 1e-9  # absolute floor (kCertScoreAbs)


def contenders(scores: np.ndarray, window: float = CERT_SCORE_REL, bounds=None) -> List[int]:
    """Candidates that can hold the fp64 maximum given certified scores: i with
    s_i >= s_b - max(e_b + e_i, window |s_b|, CERT_SCORE_ABS), e the rigorous
    per-candidate error bounds when known (Context.last_score_bounds)."""
    b = first_max(scores)
    out = []
    for i in range(len(scores)):
        e = (bounds[b] + bounds[i]) if bounds is not None else 0.0
        if scores[i] >= scores[b] - max(e, window * abs(scores[b]), CERT_SCORE_ABS):
            out.append(i)
    return out


def select_nbv_sharded(score_block: Callable[[int, int], np.ndarray], n_candidates: int, rank: int,
                       world: int, dist=None,
                       rescore: Optional[Callable[[List[int]], np.ndarray]] = None,
                       window: float = CERT_SCORE_REL) -> Tuple[int, np.ndarray]:
    """score_block(lo, hi) scores candidates [lo, hi) on this rank (certified fp32
    path). With `rescore(indices)` (exact fp64 scores of global candidate indices
    of this rank's block), every contender within `window` of the best is re-scored
    on the rank that owns it and the first-max is taken again, so the argmax is
    the fp64 one whatever the rank count (the library does the same on one GPU)."""
    lo, hi = shard_range(n_candidates, rank, world)
    local = score_block(lo, hi) if hi > lo else np.zeros(0)
    scores = gather_scores(local, n_candidates, rank, world, dist)
    if rescore is None or n_candidates == 0:
        return first_max(scores), scores
    cont = contenders(scores, window)
    if len(cont) < 2:
        return first_max(scores), scores
    mine = [i for i in cont if lo <= i < hi]
    exact = np.zeros(n_candidates)
    if mine:
        exact[mine] = np.asarray(rescore(mine), np.float64)
    if world > 1 and dist is not None:
        exact = _allreduce_sum_host(exact, dist)
    scores = scores.copy()
    scores[cont] = exact[cont]
    return first_max(scores), scores


def _allreduce_sum_host(x: np.ndarray, dist) -> np.ndarray:
    """Sum of per-rank vectors whose non-zero entries are disjoint (exact: x + 0 = x)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" \
        else torch.device("cpu")
    t = torch.as_tensor(np.asarray(x, np.float64), device=dev).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.cpu().numpy()


def construct_field_sharded(partial_field: Callable[[int, int], object], n_views: int, rank: int,
                            world: int, allreduce_sum: Callable[[object], None],
                            set_num_views: Optional[Callable[[object, int], None]] = None) -> object:
    """partial_field(lo, hi) accumulates views [lo, hi) into a fresh field and returns
    it; allreduce_sum(field) sums the partial coefficient arrays across ranks in place;
    set_num_views(field, n_views) then records the trajectory length |P| on every
    rank (construct_field sets num_views = |P|, vfield.hpp:91) -- each rank's partial
    field only counted its own block, and query_visibility uses |P| as the exponent."""
    lo, hi = shard_range(n_views, rank, world)
    field = partial_field(lo, hi)
    if world > 1:
        allreduce_sum(field)
    if set_num_views is not None:
        set_num_views(field, n_views)
    return field


def construct_device_field_sharded(ctx, scene, views: Sequence, vmf, degree: int, rank: int, world: int,
                                   dist=None, rc=None):
    """VF CONST over `views` sharded across ranks on the device: this rank
    accumulates its contiguous block (gavis_vf_accumulate_views), the fp64
    partials are summed in place by an all-reduce (NCCL over NVLink), and
    num_views is set to len(views) on every rank."""
    from . import api
    from .model import RasterConfig
    rc = rc or RasterConfig()

    def partial(lo, hi):
        f = api.empty_field(ctx, scene, vmf, degree)
        if hi > lo:
            api.accumulate_views(ctx, f, scene, views[lo:hi], rc)
        return f

    return construct_field_sharded(partial, len(views), rank, world,
                                   lambda fld: allreduce_device_field(fld, dist),
                                   lambda fld, n: fld.set_num_views(n))


class DeviceArray:
    """Exposes a raw device pointer of the native library through
    __cuda_array_interface__ so torch can alias it (zero copy) for NCCL."""

    def __init__(self, ptr: int, count: int, typestr: str = "<f8"):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def allreduce_device_field(field, dist) -> None:
    """In-place NCCL all-reduce(sum) of a DeviceField's fp64 coefficients (aliasing
    the library's device buffer); over gloo through a host copy."""
    import torch
    ptr, count = field.device_gamma()
    field.ctx.synchronize()
    t = torch.as_tensor(DeviceArray(ptr, count), device="cuda")
    if dist.get_backend() == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    else:
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM)
        t.copy_(h)
    torch.cuda.synchronize()
