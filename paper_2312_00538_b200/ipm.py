"""GPU-resident interior point SVM trainer: Python mirror of the reference's
ipm_train / compute_bias / make_model / TrainedModel
(P:include/ksvm/ipm.hpp, P:src/ipm.cpp) over an AnovaFastOperator.

    res = ipm_train(op, y, Z, IpmConfig(C=1.0))     # Z: stacked factor or None
    model = make_model(res, train, spec, FastsumConfig(), op, C=1.0)
    labels = model.predict(test_points_raw)

The loop runs in libksvm_nfft.so (ksvm_nfft_ipm_train, csrc/ipm.cu): alpha,
Theta, the Newton systems and GMRES live on the operator's GPU. Errors follow
the reference: invalid IpmConfig or labels -> ValueError
(std::invalid_argument), degenerate initial infeasibility -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .fastsum import AnovaFastOperator, AnovaKernelSpec, FastsumConfig, _is_cuda_tensor, _raise, decision_values


@dataclass
class IpmConfig:
    """P:include/ksvm/ipm.hpp:15-24 (same defaults)."""
    C: float = 0.5
    sigma: float = 0.6
    gamma0: float = 0.99995
    tol_ip: float = 1e-1
    max_ip_iters: int = 50
    tol_gmres: float = 1e-3
    max_gmres_iters: int = 100
    mu0: float = 1.0

    def _c(self) -> _lib.IpmConfig:
        return _lib.IpmConfig(float(self.C), float(self.sigma), float(self.gamma0), float(self.tol_ip),
                              int(self.max_ip_iters), float(self.tol_gmres), int(self.max_gmres_iters),
                              float(self.mu0))


class IpmStatus(enum.IntEnum):
    """P:include/ksvm/ipm.hpp:28."""
    CONVERGED = 0
    MAX_ITERATIONS = 1
    STALLED = 2


@dataclass
class GmresLog:
    iterations: int
    relative_residual: float
    converged: bool
    breakdown: bool


@dataclass
class IpmIterationLog:
    """P:include/ksvm/ipm.hpp:30-37."""
    it: int
    mu: float
    xi_alpha_rel: float
    xi_lambda_rel: float
    step_alpha: float
    gmres: GmresLog


@dataclass
class IpmResult:
    """P:include/ksvm/ipm.hpp:39-49."""
    alpha: np.ndarray
    lambda_: float
    mu_final: float
    xi_alpha_rel: float
    xi_lambda_rel: float
    status: IpmStatus
    iterations: List[IpmIterationLog] = field(default_factory=list)

    def mean_gmres_iters(self) -> float:
        if not self.iterations:
            return 0.0
        return sum(it.gmres.iterations for it in self.iterations) / len(self.iterations)


def _labels(y, n) -> np.ndarray:
    y = np.ascontiguousarray(np.asarray(y, dtype=np.float64).reshape(-1))
    if y.shape[0] != n:
        raise ValueError("ipm_train: label size mismatch")  # P:src/ipm.cpp:81
    return y


def ipm_train(op: AnovaFastOperator, y, factor=None, cfg: Optional[IpmConfig] = None) -> IpmResult:
    """ipm_train (P:src/ipm.cpp:76-155) on op's GPU. factor: the stacked
    k x n factor (stack_anova_factors) as a numpy array or a CUDA tensor on
    op's GPU (kept there), or None (unpreconditioned)."""
    cfg = cfg or IpmConfig()
    n = op.size()
    y = _labels(y, n)
    zp, k, zkind = None, 0, _lib.HOST
    if factor is not None:
        if _is_cuda_tensor(factor):
            import torch
            Zt = factor.to(torch.float64).contiguous()
            if Zt.dim() != 2 or Zt.shape[1] != n:
                raise ValueError("factor must be k x n")
            torch.cuda.current_stream(Zt.device).synchronize()  # Z complete before the library's stream reads it
            zp, k, zkind, keep = C.c_void_p(Zt.data_ptr()), int(Zt.shape[0]), _lib.DEVICE, Zt
        else:
            Z = np.ascontiguousarray(factor, dtype=np.float64)
            if Z.ndim != 2 or Z.shape[1] != n:
                raise ValueError("factor must be k x n")
            zp, k, keep = C.c_void_p(Z.ctypes.data), int(Z.shape[0]), Z
    alpha = np.empty(n)
    res = _lib.IpmResult()
    log = (_lib.IpmLog * int(max(cfg.max_ip_iters, 1)))()
    c = cfg._c()
    _raise(_lib.load().ksvm_nfft_ipm_train(op._h, C.c_void_p(y.ctypes.data), zp, k, zkind, C.byref(c),
                                           C.c_void_p(alpha.ctypes.data), C.byref(res), log))
    its = [IpmIterationLog(L.it, L.mu, L.xi_alpha_rel, L.xi_lambda_rel, L.step_alpha,
                           GmresLog(L.gmres_iterations, L.gmres_relative_residual, bool(L.gmres_converged),
                                    bool(L.gmres_breakdown)))
           for L in log[: res.iterations]]
    return IpmResult(alpha, float(res.lambda_), float(res.mu_final), float(res.xi_alpha_rel),
                     float(res.xi_lambda_rel), IpmStatus(res.status), its)


def compute_bias(alpha, y, op: AnovaFastOperator, C_: float, eps_sv: float) -> float:
    """compute_bias (P:src/ipm.cpp:157-185)."""
    n = op.size()
    a = np.ascontiguousarray(np.asarray(alpha, dtype=np.float64).reshape(-1))
    y = _labels(y, n)
    if a.shape[0] != n:
        raise ValueError("compute_bias: size mismatch")
    b = C.c_double(0.0)
    _raise(_lib.load().ksvm_nfft_compute_bias(op._h, C.c_void_p(a.ctypes.data), C.c_void_p(y.ctypes.data),
                                              float(C_), float(eps_sv), C.byref(b), None))
    return float(b.value)


def dual_objective(alpha, y, op: AnovaFastOperator) -> float:
    """SVM dual objective 1^T alpha - 1/2 alpha^T Y K Y alpha at the
    operator's kernel (the quantity the IPM maximises)."""
    a = np.asarray(alpha, dtype=np.float64)
    ya = np.asarray(y, dtype=np.float64) * a
    return float(a.sum() - 0.5 * ya @ op.apply(ya))


@dataclass
class FeatureStats:
    """P:include/ksvm/dataset.hpp:19-22."""
    mean: float = 0.0
    stddev: float = 1.0


def apply_normalization(points, stats) -> np.ndarray:
    """P:src/dataset.cpp:284-295."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.shape[1] != len(stats):
        raise ValueError("dimension mismatch in normalization")
    out = pts.copy()
    for j, s in enumerate(stats):
        out[:, j] = (out[:, j] - s.mean) / s.stddev
    return out


@dataclass
class TrainedModel:
    """P:include/ksvm/ipm.hpp:53-71."""
    alpha: np.ndarray
    bias: float
    y: np.ndarray
    train_points: np.ndarray   # normalized coordinates
    kernel: AnovaKernelSpec
    normalization: list
    fastsum: FastsumConfig
    support_indices: np.ndarray
    dual_feasibility: float
    device: int = 0

    def decision_values(self, test_points, backend: str = "fast") -> np.ndarray:
        """f(x) for raw (unnormalized) test points (P:src/ipm.cpp:213-288), on the GPU."""
        pts = np.asarray(test_points, dtype=np.float64)
        if pts.shape[1] != self.train_points.shape[1]:
            raise ValueError("predict: feature dimension mismatch")
        if self.normalization:
            pts = apply_normalization(pts, self.normalization)
        f, _ = decision_values(self.train_points, self.kernel, self.alpha * self.y, self.bias, pts, backend,
                               self.fastsum, self.device)
        return f

    def predict(self, test_points, backend: str = "fast") -> np.ndarray:
        """sign(f(x)) with sign(0) = +1 (P:src/ipm.cpp:290-294)."""
        return np.where(self.decision_values(test_points, backend) >= 0.0, 1.0, -1.0)


def make_model(result: IpmResult, train, spec: AnovaKernelSpec, fs: FastsumConfig, op: AnovaFastOperator,
               C_: float, normalization=None) -> TrainedModel:
    """make_model (P:src/ipm.cpp:187-211)."""
    eps_sv = 1e-4 * C_
    y = np.asarray(train.labels, dtype=np.float64)
    bias = compute_bias(result.alpha, y, op, C_, eps_sv)
    sv = np.nonzero(result.alpha > eps_sv)[0]
    return TrainedModel(result.alpha.copy(), bias, y.copy(), np.asarray(train.points, dtype=np.float64).copy(), spec,
                        list(normalization or []), fs, sv, float(abs(y @ result.alpha)), op.device)
