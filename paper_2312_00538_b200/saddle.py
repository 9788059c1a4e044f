"""GPU-resident Newton saddle solver: Python mirror of the
reference's SaddleOperator / SaddlePreconditioner / gmres_solve
(P:include/ksvm/saddle.hpp, P:src/saddle.cpp) over an AnovaFastOperator.

    op = SaddleOperator(K, y, theta)          # K: AnovaFastOperator
    P = SaddlePreconditioner(Z, y)            # Z: k x n stacked factor or None
    P.refresh(theta)
    x, stats = gmres_solve(op, P, rhs, tol, max_iter)

Vectors have n + 1 entries; numpy arrays run through host copies, CUDA torch
tensors stay on the device (torch's current stream). Errors follow the
reference: non-positive Theta / tol -> ValueError, apply before refresh ->
RuntimeError (std::logic_error).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .fastsum import AnovaFastOperator, _raise, _Vec


def _host(a, n=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1))
    if n is not None and a.shape[0] != n:
        raise ValueError("length mismatch")
    return a


class SaddleOperator:
    """[Y K Y + Theta, -y; -y^T, 0] (P:include/ksvm/saddle.hpp:14-31)."""

    def __init__(self, op: AnovaFastOperator, y, theta):
        n = op.size()
        self.op, self.n = op, n
        self.device = op.device
        self._y = _host(y, n)
        h = C.c_void_p()
        _raise(_lib.load().ksvm_nfft_saddle_create(op._h, C.c_void_p(self._y.ctypes.data),
                                                   C.c_void_p(_host(theta, n).ctypes.data), C.byref(h)))
        self._h = h
        self._free = _lib.load().ksvm_nfft_saddle_free

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    def size(self) -> int:
        return self.n + 1

    def set_theta(self, theta) -> None:
        _raise(_lib.load().ksvm_nfft_saddle_set_theta(self._h, C.c_void_p(_host(theta, self.n).ctypes.data)))

    def apply(self, vw):
        a = _Vec(vw, self.n + 1, self.device)
        out, po = a.out(self.n + 1)
        _raise(_lib.load().ksvm_nfft_saddle_apply(self._h, a.ptr, po, a.kind, a.stream))
        return out


class SaddlePreconditioner:
    """Block-triangular SMW preconditioner (P:include/ksvm/saddle.hpp:33-58).
    Z None: identity (a null StackedFactor)."""

    def __init__(self, Z, y, device: int = 0):
        y = _host(y)
        self.n = y.shape[0]
        self.device = int(device)
        Zc = None if Z is None else np.ascontiguousarray(Z, dtype=np.float64)
        if Zc is not None and (Zc.ndim != 2 or Zc.shape[1] != self.n):
            raise ValueError("Z must be k x n")
        h = C.c_void_p()
        _raise(_lib.load().ksvm_nfft_precond_create(None if Zc is None else C.c_void_p(Zc.ctypes.data),
                                                    0 if Zc is None else Zc.shape[0], self.n,
                                                    C.c_void_p(y.ctypes.data), self.device, C.byref(h)))
        self._h = h
        self._free = _lib.load().ksvm_nfft_precond_free

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    def refresh(self, theta) -> None:
        _raise(_lib.load().ksvm_nfft_precond_refresh(self._h, C.c_void_p(_host(theta, self.n).ctypes.data)))

    def apply(self, g):
        a = _Vec(g, self.n + 1, self.device)
        out, po = a.out(self.n + 1)
        _raise(_lib.load().ksvm_nfft_precond_apply(self._h, a.ptr, po, a.kind, a.stream))
        return out

    def identity(self) -> bool:
        return bool(_lib.load().ksvm_nfft_precond_identity(self._h))

    def diagonal_fallback(self) -> bool:
        return bool(_lib.load().ksvm_nfft_precond_diagonal_fallback(self._h))


@dataclass
class GmresStats:
    """P:include/ksvm/saddle.hpp:60-66."""
    iterations: int = 0
    relative_residual: float = 0.0
    converged: bool = False
    breakdown: bool = False
    residual_history: list = field(default_factory=list)


def gmres_solve(op: SaddleOperator, precond: SaddlePreconditioner, rhs, tol: float, max_iter: int):
    """Right-preconditioned full GMRES, x0 = 0 (P:src/saddle.cpp:92-178).
    Returns (x, GmresStats)."""
    a = _Vec(rhs, op.n + 1, op.device)
    out, po = a.out(op.n + 1)
    st = _lib.GmresStats()
    hist = np.zeros(max(int(max_iter), 1))
    _raise(_lib.load().ksvm_nfft_gmres_solve(op._h, precond._h, a.ptr, float(tol), int(max_iter), po, C.byref(st),
                                             C.c_void_p(hist.ctypes.data), a.kind, a.stream))
    return out, GmresStats(int(st.iterations), float(st.relative_residual), bool(st.converged), bool(st.breakdown),
                           list(hist[:st.iterations]))
