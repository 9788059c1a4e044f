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


def pipelined_matvec(op, v, y, chunks: int, allreduce_async: Callable) -> None:
    """Window-sharded matvec with the cross-rank sum chunked and overlapped
    (SURVEY.md 8(e) "chunk it and overlap"): the rank's windows run first
    (``op.apply_windows``), then for each of `chunks` row ranges the window
    sum of that range is launched and its all-reduce issued asynchronously,
    so range k is on the wire while range k+1 is being summed. `op` is a
    window-masked AnovaFastOperator, v / y CUDA tensors of length n;
    ``allreduce_async(t)`` returns a handle with ``wait()`` (torch.distributed
    ``all_reduce(..., async_op=True)``). Returns after every handle is waited."""
    n = y.numel()
    op.apply_windows(v)
    handles = []
    for k in range(chunks):
        lo, hi = n * k // chunks, n * (k + 1) // chunks
        if hi > lo:
            op.combine_range(y, lo, hi)
            handles.append(allreduce_async(y[lo:hi]))
    for h in handles:
        h.wait()


class _Done:
    def wait(self):
        return None


def make_collectives(backend: str):
    """(allreduce, allreduce_async, allgather) on the default process group
    for CUDA tensors. "nccl": the NCCL collectives in place on the device
    (NVLink / NVSwitch); "gloo": staged through host memory -- used to run the
    multi-rank path on a single GPU (ranks sharing one device) and in tests;
    its "async" all-reduce completes before returning."""
    import torch
    import torch.distributed as dist
    if backend == "nccl":
        def allreduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

        def allreduce_async(t):
            return dist.all_reduce(t, op=dist.ReduceOp.SUM, async_op=True)

        def allgather(out, inp):
            dist.all_gather_into_tensor(out, inp)
        return allreduce, allreduce_async, allgather

    def allreduce(t):
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
        t.copy_(c)

    def allreduce_async(t):
        allreduce(t)
        return _Done()

    def allgather(out, inp):
        c = inp.cpu()
        parts = [torch.empty_like(c) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, c)
        out.copy_(torch.cat(parts))
    return allreduce, allreduce_async, allgather


def torch_allreduce(t) -> None:
    import torch.distributed as dist
    dist.all_reduce(t, op=dist.ReduceOp.SUM)


def numpy_allreduce_via_torch(a: np.ndarray) -> None:
    """In-place sum of a numpy vector over the default group (gloo on CPU)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(a)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)


# ---- point sharding (SURVEY.md 8(e) hybrid: balance independent of P) -------

def point_shard(n: int, world: int, rank: int) -> np.ndarray:
    """Owned rows of `rank`: a contiguous block of the n points (sizes differ
    by at most one)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return np.arange(lo, hi, dtype=np.int64)


def point_block(n: int, world: int, rank: int) -> np.ndarray:
    """Owned rows of `rank` in blocks of ceil(n / world) rows (the last one
    shorter), so the output can be assembled with one all-gather of equal
    blocks: rank r's rows are [r b, min(n, (r + 1) b)), b = ceil(n / world)."""
    b = -(-n // world)
    return np.arange(min(n, rank * b), min(n, (rank + 1) * b), dtype=np.int64)


class _DevView:
    """__cuda_array_interface__ view of library-owned device memory (zero copy)."""

    def __init__(self, ptr: int, length: int):
        self.__cuda_array_interface__ = {"shape": (int(length),), "typestr": "<f8", "data": (int(ptr), False),
                                          "version": 3}


class PointShardedOperator:
    """One rank's share of a point-sharded ANOVA operator
    (ksvm_nfft_op_create_sharded): planned from all n points, spreading and
    gathering only `own_points`. A matvec is

        op.apply_spread(v)                 # owned points -> per-window grids
        for g in op.grids(): allreduce(g)  # sum the partial grids over ranks
        op.apply_finish(y)                 # owned rows of y, zeros elsewhere
        allreduce(y)                       # full y on every rank

    (``matvec(v, y, allreduce)`` does exactly that). v and y are CUDA tensors
    on the operator's device (torch's current stream) or numpy arrays."""

    def __init__(self, data, spec, own_points, cfg=None, fit_fraction: float = 1.0, device: int = 0,
                 precision: str = "fp64"):
        import ctypes as C
        from . import _lib
        from .fastsum import FastsumConfig, _host_matrix, _precision, _raise
        cfg = cfg or FastsumConfig()
        a = _host_matrix(data.points if hasattr(data, "points") else data)
        n, d = a.shape
        w = spec.windowing
        P = w.num_windows()
        feats = (C.c_int * max(1, sum(len(x) for x in w.windows)))(*[int(f) for x in w.windows for f in x])
        sizes = (C.c_int * max(1, P))(*[len(x) for x in w.windows])
        eta = (C.c_double * max(1, P))(*[float(x) for x in w.weights])
        ell = (C.c_double * max(1, P))(*[float(x) for x in w.length_scales])
        own = np.ascontiguousarray(np.asarray(own_points, dtype=np.int64))
        c = cfg._c()
        h = C.c_void_p()
        _raise(_lib.load().ksvm_nfft_op_create_sharded(C.c_void_p(a.ctypes.data), n, d, d, _lib.ROW_MAJOR, feats, sizes,
                                                       P, eta, ell, C.byref(c), float(fit_fraction),
                                                       C.c_void_p(own.ctypes.data), own.shape[0], int(device),
                                                       _precision(precision), C.byref(h)))
        self._h, self._n, self.device, self.own = h, n, int(device), own
        self._free = _lib.load().ksvm_nfft_op_free

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    def size(self) -> int:
        return self._n

    def _io(self, x, n):
        import ctypes as C
        from . import _lib
        try:
            import torch
            if isinstance(x, torch.Tensor) and x.is_cuda:
                if x.dtype != torch.float64 or not x.is_contiguous() or x.numel() != n:
                    raise ValueError("expected a contiguous float64 CUDA tensor of length n")
                return C.c_void_p(x.data_ptr()), _lib.DEVICE, C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
        except ImportError:
            pass
        if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous and x.size == n):
            raise ValueError("expected a contiguous float64 array of length n")
        return C.c_void_p(x.ctypes.data), _lib.HOST, C.c_void_p(0)

    def apply_spread(self, v) -> None:
        from . import _lib
        from .fastsum import _raise
        p, kind, st = self._io(v, self._n)
        _raise(_lib.load().ksvm_nfft_op_apply_spread(self._h, p, kind, st))

    def grids(self):
        """The per-window grids G (CUDA tensor views, window order)."""
        import ctypes as C
        import torch
        from . import _lib
        cnt = _lib.load().ksvm_nfft_op_grids(self._h, None, None, 0)
        if cnt < 0:
            from .fastsum import _raise
            _raise(-cnt)
        ptrs = (C.c_void_p * max(cnt, 1))()
        lens = (C.c_int64 * max(cnt, 1))()
        _lib.load().ksvm_nfft_op_grids(self._h, ptrs, lens, cnt)
        dev = torch.device("cuda", self.device)
        return [torch.as_tensor(_DevView(ptrs[k], lens[k]), device=dev) for k in range(cnt)]

    def grid_pool(self):
        """The owned windows' grids G as ONE contiguous CUDA tensor view
        (ksvm_nfft_op_grid_pool): one all-reduce per matvec sums them."""
        import ctypes as C
        import torch
        from . import _lib
        from .fastsum import _raise
        p, ln = C.c_void_p(), C.c_int64()
        _raise(_lib.load().ksvm_nfft_op_grid_pool(self._h, C.byref(p), C.byref(ln)))
        return torch.as_tensor(_DevView(p.value, ln.value), device=torch.device("cuda", self.device))

    def apply_finish(self, y) -> None:
        from . import _lib
        from .fastsum import _raise
        p, kind, st = self._io(y, self._n)
        _raise(_lib.load().ksvm_nfft_op_apply_finish(self._h, p, kind, st))

    def matvec(self, v, y, allreduce: Callable = None) -> None:
        self.apply_spread(v)
        if allreduce is not None:
            allreduce(self.grid_pool())
        self.apply_finish(y)
        if allreduce is not None:
            allreduce(y)

    def matvec_blocks(self, v, y_pad, rank: int, world: int, allreduce: Callable, allgather: Callable) -> None:
        """Matvec for point_block shards: grids summed with one all-reduce,
        y assembled with one all-gather of the equal row blocks (half the
        bytes of an all-reduce of y). y_pad: CUDA tensor of world * ceil(n /
        world) entries; y_pad[:n] is the product afterwards.
        ``allgather(out, inp)`` gathers equal blocks into out."""
        n = self._n
        b = -(-n // world)
        self.apply_spread(v)
        allreduce(self.grid_pool())
        y = y_pad[:n]
        self.apply_finish(y)
        blk = y_pad[rank * b:(rank + 1) * b].clone()
        allgather(y_pad, blk)
