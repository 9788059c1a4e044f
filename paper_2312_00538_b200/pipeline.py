"""End-to-end training on the B200 path: Python mirror of the reference's
pipeline (P:include/ksvm/pipeline.hpp, P:src/pipeline.cpp) for the parts
that reach the hot path:

    model, test, report = train_pipeline(Dataset(X, y), PipelineConfig(
        explicit_windows=[[0, 1, 2], [3, 4, 5]], rank=50, ipm=IpmConfig(C=1.0)))
    acc = (model.predict(test_raw_points) == test.labels).mean()

balance_and_split -> zscore_fit_transform -> explicit windows (eta = 1/P,
ell = 1) -> GPU greedy pivoted-Cholesky factor per window, stacked with
sqrt(eta) -> GPU interior point loop over the NFFT operator (fit 1/1.2) ->
compute_bias -> TrainedModel (GPU prediction). Nystrom factors (columns /
Gaussian sketch) are built on the GPU too; mutual-information windowing,
random-pivot Cholesky and random Fourier features are outside this path
(DESIGN.md).
"""
from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field
from typing import List

import numpy as np
import torch

from . import _lib
from .fastsum import (AnovaKernelSpec, Dataset, FastsumConfig, FeatureWindowing, _raise, anova_fast_operator)
from .ipm import FeatureStats, IpmConfig, IpmStatus, ipm_train, make_model
from .lowrank import fast_window_operator, nystrom, pivoted_cholesky_greedy, stack_anova_factors

PRECOND_METHODS = ("none", "cholesky-greedy", "nystrom-columns", "nystrom-gaussian")  # P:src/pipeline.cpp:8-18


@dataclass
class PipelineConfig:
    """P:include/ksvm/pipeline.hpp:32-47 (defaults kept)."""
    train_fraction: float = 0.5
    seed: int = 0
    explicit_windows: list = field(default_factory=list)   # [[0, 1, 2], [3, 4]] (0-based)
    length_scales: list = field(default_factory=list)      # empty = 1 per window; 1 entry = shared
    precond: str = "cholesky-greedy"
    rank: int = 200
    per_window_ranks: list = field(default_factory=list)
    cholesky_err_tol: float = 1e-5
    fastsum: FastsumConfig = field(default_factory=FastsumConfig)
    ipm: IpmConfig = field(default_factory=IpmConfig)
    device: int = 0


@dataclass
class TrainReport:
    """P:include/ksvm/pipeline.hpp:49-63."""
    n_train: int = 0
    n_test: int = 0
    d: int = 0
    P: int = 0
    rank: int = 0
    fit_seconds: float = 0.0
    precond_setup_seconds: float = 0.0
    ipm_iters: int = 0
    mean_gmres: float = 0.0
    xi_alpha: float = 0.0
    xi_lambda: float = 0.0
    mu_final: float = 0.0
    status: IpmStatus = IpmStatus.CONVERGED
    phase_seconds: dict = field(default_factory=dict)  # (addition) operator / factor / ipm / model wall times


def parse_window_spec(spec: str, d: int) -> List[List[int]]:
    """P:src/pipeline.cpp:28-52: "0,1,2;3,4" -> [[0, 1, 2], [3, 4]]."""
    windows = []
    for group in spec.split(";"):
        win = []
        for item in group.split(","):
            if not item:
                continue
            try:
                f = int(item)
            except ValueError:
                raise ValueError(f"bad window spec item: '{item}'") from None
            if f < 0 or f >= d:
                raise ValueError(f"window feature index out of range: {item}")
            win.append(f)
        if win:
            windows.append(win)
    if not windows:
        raise ValueError(f"window spec has no windows: '{spec}'")
    return windows


def balance_and_split(data: Dataset, train_fraction: float = 0.5, seed: int = 0):
    """balance_and_split (P:src/dataset.cpp:212-262): the reference's
    std::mt19937_64 / std::shuffle stream (libksvm_nfft.so), so the split is
    the reference's. Returns (train, test) Datasets."""
    lab = np.ascontiguousarray(np.asarray(data.labels, dtype=np.float64).reshape(-1))
    n = lab.shape[0]
    tr = np.zeros(max(n, 1), dtype=np.int64)
    te = np.zeros(max(n, 1), dtype=np.int64)
    ntr, nte = C.c_int64(0), C.c_int64(0)
    _raise(_lib.load().ksvm_nfft_balance_and_split(C.c_void_p(lab.ctypes.data), n, float(train_fraction), int(seed),
                                                   C.c_void_p(tr.ctypes.data), C.byref(ntr),
                                                   C.c_void_p(te.ctypes.data), C.byref(nte)))
    tr, te = tr[: ntr.value], te[: nte.value]
    pts = torch.from_numpy(np.ascontiguousarray(data.points, dtype=np.float64))
    rows = lambda idx: torch.index_select(pts, 0, torch.from_numpy(idx)).numpy()  # threaded exact row copy
    return Dataset(rows(tr), lab[tr]), Dataset(rows(te), lab[te])


def zscore_fit_transform(train: Dataset, test: Dataset):
    """zscore_fit_transform (P:src/dataset.cpp:264-282): per-feature mean and
    population standard deviation of the training part (sd < 1e-300 -> 1),
    applied to both parts. Returns the FeatureStats list."""
    if train.n() == 0:
        raise ValueError("empty training split")
    # sums in numpy (fixed order), elementwise passes on torch's CPU threads
    # (exact: the same IEEE operations per element)
    Xt = torch.from_numpy(np.ascontiguousarray(train.points, dtype=np.float64)).clone()
    X = Xt.numpy()
    n = X.shape[0]
    mean = X.sum(axis=0) / n
    Xt.sub_(torch.from_numpy(mean))
    sd = np.sqrt(torch.mul(Xt, Xt).numpy().sum(axis=0) / n)  # = ((X - mean) ** 2).sum(0) / n
    sd[sd < 1e-300] = 1.0  # constant column maps to zeros
    Xt.div_(torch.from_numpy(sd))
    train.points = X
    if test is not None and test.n() > 0:
        Tt = torch.from_numpy(np.ascontiguousarray(test.points, dtype=np.float64)).clone()
        Tt.sub_(torch.from_numpy(mean)).div_(torch.from_numpy(sd))
        test.points = Tt.numpy()
    return [FeatureStats(float(a), float(b)) for a, b in zip(mean, sd)]


def window_ranks(cfg: PipelineConfig, P: int, n: int) -> List[int]:
    """P:src/pipeline.cpp:73-86."""
    if cfg.per_window_ranks:
        if len(cfg.per_window_ranks) != P:
            raise ValueError("per_window_ranks size must equal P")
        ranks = list(cfg.per_window_ranks)
    else:
        ranks = [max(1, cfg.rank // P)] * P
    return [min(int(r), n) for r in ranks]


def build_precond_factor(op, train: Dataset, spec: AnovaKernelSpec, cfg: PipelineConfig, on_device: bool = False):
    """build_precond_factor (P:src/pipeline.cpp:137-196): one factor per
    window on the GPU, stacked with sqrt(eta_l) (stack_anova_factors,
    P:src/low_rank.cpp:200-222). cholesky-greedy and nystrom-columns use the
    window's exact kernel (WindowOperator); nystrom-gaussian sketches the
    window's FastWindowOperator (a one-window NFFT operator, fit 1.0) with
    seed cfg.seed + l. on_device keeps every factor and the stack in HBM (a
    CUDA tensor; the IPM's preconditioner then never crosses PCIe). Returns
    (Z k x n, setup seconds)."""
    if cfg.precond not in PRECOND_METHODS[1:]:
        raise ValueError(f"preconditioner '{cfg.precond}' is not on the B200 path "
                         f"(supported: {', '.join(PRECOND_METHODS)})")
    w = spec.windowing
    P = w.num_windows()
    ranks = window_ranks(cfg, P, train.n())
    t0 = time.perf_counter()
    factors = []
    if cfg.precond == "nystrom-gaussian":
        # The sketch draws (the reference's sequential libstdc++ normal stream,
        # seed + l) dominate on the host; windows are independent, so their
        # factors are built concurrently (ctypes releases the GIL; each window
        # has its own operator and stream).
        from concurrent.futures import ThreadPoolExecutor
        if on_device:
            import torch
            torch.cuda.current_stream(torch.device("cuda", op.device)).synchronize()

        def one(l):  # the window's FastWindowOperator (its own plan) and its sketch
            if on_device:
                import torch
                torch.cuda.set_device(op.device)
            fop = fast_window_operator(train.points, w.windows[l], w.length_scales[l], cfg.fastsum, op.device)
            return nystrom(fop, ranks[l], "gaussian", int(cfg.seed) + l, on_device=on_device)

        with ThreadPoolExecutor(max_workers=max(1, min(P, os.cpu_count() or 1))) as ex:
            factors = list(ex.map(one, range(P)))
        if on_device:
            import torch
            torch.cuda.synchronize(op.device)
    for l in range(P if cfg.precond != "nystrom-gaussian" else 0):
        seed = int(cfg.seed) + l
        if cfg.precond == "cholesky-greedy":
            f = pivoted_cholesky_greedy(op, ranks[l], cfg.cholesky_err_tol, window=l, on_device=on_device)
        else:
            f = nystrom(op, ranks[l], "columns", seed, window=l, on_device=on_device)
        factors.append(f)
    if on_device:
        import torch
        Z = torch.cat([f.Z * float(np.sqrt(wt)) for f, wt in zip(factors, w.weights)], dim=0)
        torch.cuda.current_stream(Z.device).synchronize()
    else:
        Z = stack_anova_factors(factors, w.weights)
    return Z, time.perf_counter() - t0


def train_on_prepared(train: Dataset, spec: AnovaKernelSpec, cfg: PipelineConfig, report: TrainReport,
                      normalization=None):
    """train_on_prepared (P:src/pipeline.cpp:198-227) with the fast backend:
    returns (TrainedModel, IpmResult)."""
    t0 = time.perf_counter()
    op = anova_fast_operator(train, spec, cfg.fastsum, 1.0 / 1.2, device=cfg.device)
    t1 = time.perf_counter()
    Z = None
    if cfg.precond != "none":
        Z, report.precond_setup_seconds = build_precond_factor(op, train, spec, cfg, on_device=True)
    t2 = time.perf_counter()
    res = ipm_train(op, train.labels, Z, cfg.ipm)
    t3 = time.perf_counter()
    model = make_model(res, train, spec, cfg.fastsum, op, cfg.ipm.C, normalization)
    report.phase_seconds = {"operator": t1 - t0, "factor": t2 - t1, "ipm": t3 - t2,
                            "model": time.perf_counter() - t3}
    report.n_train = train.n()
    report.d = train.dim()
    report.P = spec.windowing.num_windows()
    report.rank = 0 if Z is None else int(Z.shape[0])
    report.fit_seconds = time.perf_counter() - t0
    report.ipm_iters = len(res.iterations)
    report.mean_gmres = res.mean_gmres_iters()
    report.xi_alpha = res.xi_alpha_rel
    report.xi_lambda = res.xi_lambda_rel
    report.mu_final = res.mu_final
    report.status = res.status
    return model, res


def train_pipeline(raw: Dataset, cfg: PipelineConfig):
    """train_pipeline (P:src/pipeline.cpp:229-265) with explicit windows:
    returns (TrainedModel, normalized test Dataset, TrainReport, IpmResult)."""
    t0 = time.perf_counter()
    train, test = balance_and_split(raw, cfg.train_fraction, cfg.seed)
    stats = zscore_fit_transform(train, test)
    t_prep = time.perf_counter() - t0
    if not cfg.explicit_windows:
        raise ValueError("mutual-information windowing is outside the B200 path: pass explicit_windows")
    windows = cfg.explicit_windows
    if isinstance(windows, str):
        windows = parse_window_spec(windows, train.dim())
    for win in windows:
        for f in win:
            if f < 0 or f >= train.dim():
                raise ValueError(f"window feature index out of range: {f}")
    wnd = FeatureWindowing.explicit(windows)
    if cfg.length_scales:
        P = wnd.num_windows()
        if len(cfg.length_scales) == 1:
            wnd.length_scales = [float(cfg.length_scales[0])] * P
        elif len(cfg.length_scales) == P:
            wnd.length_scales = [float(x) for x in cfg.length_scales]
        else:
            raise ValueError("length_scales must have 1 or P entries")
    spec = AnovaKernelSpec(wnd)
    report = TrainReport()
    model, res = train_on_prepared(train, spec, cfg, report, stats)
    report.phase_seconds["split_zscore"] = t_prep
    report.n_test = test.n()
    return model, test, report, res
