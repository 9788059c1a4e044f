"""Multi-GPU window sharding of the ANOVA matvec.

Windows are independent; each rank owns a subset (LPT on the per-point cost
(2m)^{d_l}), computes the partial sum over its windows on its own GPU, and
one all-reduce (sum, fp64, length n) over NCCL / NVLink completes
y = sum_l eta_l K~_l v. The all-reduce is the only data-path collective.
"""
from __future__ import annotations

from typing import Callable, List, Sequence

import numpy as np


DEDUP_RATIO = 8  # = kDedupRatio in nfft_capi.cu


def evaluated_points(points: np.ndarray, window: Sequence[int]) -> int:
    """Points a window is evaluated on: n, or its distinct tuples when the
    library's exact duplicate merge applies (>= DEDUP_RATIO-fold shrink;
    same 4096-point sample test as find_duplicates in nfft_capi.cu)."""
    x = np.ascontiguousarray(points[:, list(window)])
    n = x.shape[0]
    s = x[:4096]
    if len(np.unique(s, axis=0)) * DEDUP_RATIO > len(s) or n < 2 * DEDUP_RATIO:
        return n
    u = len(np.unique(x, axis=0))
    return u if u * DEDUP_RATIO <= n else n


def window_costs(windows: Sequence[Sequence[int]], m: int = 4, points: np.ndarray = None) -> List[int]:
    """Spread+gather cost of each window, 2 (2m)^{d_l} FMA per evaluated
    point (per point of the dataset when `points` is not given)."""
    if points is None:
        return [2 * (2 * m) ** len(w) for w in windows]
    return [2 * (2 * m) ** len(w) * evaluated_points(points, w) for w in windows]


def lpt_assign(costs: Sequence[float], world: int) -> List[int]:
    """Longest-processing-time-first: owner rank of each window.

    Deterministic: ties broken by window index, then by lowest rank."""
    order = sorted(range(len(costs)), key=lambda l: (-costs[l], l))
    load = [0.0] * world
    owner = [0] * len(costs)
    for l in order:
        r = min(range(world), key=lambda k: (load[k], k))
        owner[l] = r
        load[r] += costs[l]
    return owner


def window_mask(owner: Sequence[int], rank: int) -> List[bool]:
    return [o == rank for o in owner]


class ShardedAnovaOperator:
    """y = allreduce_sum(partial_rank(v)); partial_rank sums the rank's windows.

    ``make_local(mask)`` builds the rank-local operator over the owned windows
    (on a GPU: ``anova_fast_operator(..., window_mask=mask)``); ``allreduce``
    sums a vector over the group in place (torch.distributed on NCCL for
    CUDA tensors, gloo for the CPU tests)."""

    def __init__(self, windows, rank: int, world: int, make_local: Callable, allreduce: Callable,
                 m: int = 4):
        self.owner = lpt_assign(window_costs(windows, m), world)
        self.mask = window_mask(self.owner, rank)
        self.rank, self.world = rank, world
        self.local = make_local(self.mask)
        self._allreduce = allreduce

    def apply(self, v):
        y = self.local.apply(v)
        self._allreduce(y)
        return y

    def owned_windows(self) -> List[int]:
        return [l for l, o in enumerate(self.owner) if o == self.rank]


def torch_allreduce(t) -> None:
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM)


def numpy_allreduce_via_torch(a: np.ndarray) -> None:
    """In-place sum of a numpy vector over the default group (gloo on CPU)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(a)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
