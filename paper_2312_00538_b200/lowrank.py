"""GPU greedy pivoted Cholesky: Python mirror of the
reference's pivoted_cholesky_greedy (P:include/ksvm/low_rank.hpp,
P:src/low_rank.cpp:25-92) on an AnovaFastOperator's exact entries.

    f = pivoted_cholesky_greedy(op, rank, err_tol, window=l)   # WindowOperator(l)
    f = pivoted_cholesky_greedy(op, rank, err_tol)             # the ANOVA kernel
    f.Z (achieved_rank x n), f.achieved_rank, f.trace_residual, f.pivots

The factor of window l is what the IPM stacks with sqrt(eta_l)
(stack_anova_factors, P:src/low_rank.cpp:200-222) into the Z of
SaddlePreconditioner.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .fastsum import AnovaFastOperator, _raise


@dataclass
class LowRankFactor:
    """P:include/ksvm/low_rank.hpp LowRankFactor (+ the pivot sequence)."""
    Z: np.ndarray
    method: str
    achieved_rank: int
    trace_residual: float
    pivots: np.ndarray


def pivoted_cholesky_greedy(op: AnovaFastOperator, rank: int, err_tol: float = 0.0, window: int = -1,
                            on_device: bool = False):
    """on_device=True keeps Z on the operator's GPU (a CUDA torch tensor,
    ordered on torch's current stream), e.g. for SaddlePreconditioner."""
    n = op.size()
    rr = max(1, min(int(rank), n))
    piv = np.zeros(rr, dtype=np.int64)
    r = C.c_int(0)
    tr = C.c_double(0.0)
    if on_device:
        import torch
        Z = torch.empty((rr, n), dtype=torch.float64, device=f"cuda:{op.device}")
        kind, stream = _lib.DEVICE, C.c_void_p(torch.cuda.current_stream(Z.device).cuda_stream)
        zp = C.c_void_p(Z.data_ptr())
    else:
        Z = np.empty((rr, n))
        kind, stream, zp = _lib.HOST, C.c_void_p(0), C.c_void_p(Z.ctypes.data)
    _raise(_lib.load().ksvm_nfft_pivoted_cholesky(op._h, int(window), int(rank), float(err_tol), zp, C.byref(r),
                                                  C.byref(tr), C.c_void_p(piv.ctypes.data), kind, stream))
    k = r.value
    return LowRankFactor(Z[:k], "cholesky-greedy", k, tr.value, piv[:k].copy())


def stack_anova_factors(factors, weights) -> np.ndarray:
    """sqrt(eta_l) Z_l stacked in window order (P:src/low_rank.cpp:200-222)."""
    if not factors or len(factors) != len(weights):
        raise ValueError("stack_anova_factors: size mismatch")
    return np.vstack([np.sqrt(w) * f.Z for f, w in zip(factors, weights)])


NYSTROM_COLUMNS, NYSTROM_GAUSSIAN = 0, 1


def nystrom(op: AnovaFastOperator, rank: int, mode: str, seed: int, ldl_threshold: float = 1e-8, window: int = -1,
            on_device: bool = False):
    """nystrom(op, rank, mode, seed, ldl_threshold) (P:src/low_rank.cpp:115-168).
    mode "gaussian" sketches op's own NFFT applies (window -1; the reference
    uses a one-window FastWindowOperator, see fast_window_operator); mode
    "columns" samples exact kernel columns of `window` (-1: ANOVA entries).
    Returns a LowRankFactor (Z: rank x n)."""
    m = {"columns": NYSTROM_COLUMNS, "gaussian": NYSTROM_GAUSSIAN}[mode]
    n = op.size()
    k = int(rank)
    if on_device:
        import torch
        Z = torch.empty((max(k, 1), n), dtype=torch.float64, device=f"cuda:{op.device}")
        kind, stream = _lib.DEVICE, C.c_void_p(torch.cuda.current_stream(Z.device).cuda_stream)
        zp = C.c_void_p(Z.data_ptr())
    else:
        Z = np.empty((max(k, 1), n))
        kind, stream, zp = _lib.HOST, C.c_void_p(0), C.c_void_p(Z.ctypes.data)
    _raise(_lib.load().ksvm_nfft_nystrom(op._h, int(window), k, m, int(seed), float(ldl_threshold), zp, kind, stream))
    return LowRankFactor(Z[:k], "nystrom-" + mode, k, 0.0, np.zeros(0, dtype=np.int64))


def fast_window_operator(points, window, length_scale: float, cfg=None, device: int = 0) -> AnovaFastOperator:
    """FastWindowOperator (P:src/pipeline.cpp:114-133): the fast transform of
    one window (weight 1, plan fit 1.0) as an operator."""
    from .fastsum import AnovaKernelSpec, FeatureWindowing, anova_fast_operator
    spec = AnovaKernelSpec(FeatureWindowing([list(window)], [1.0], [float(length_scale)], []))
    return anova_fast_operator(points, spec, cfg, 1.0, device=device)
