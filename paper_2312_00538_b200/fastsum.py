"""Reference-facing host API of the B200 NFFT fast summation.

Mirrors the reference's operator seam for this path (names, argument
meaning, error behaviour) so that callers and tests read like the
reference's own:

=============================  =================================================
this module                    reference (P: = /root/reference/proj)
=============================  =================================================
FastsumConfig                  P:include/ksvm/fastsum.hpp:13-20, validate :38-47
GaussianKernelSpec             P:include/ksvm/kernel.hpp:11-13
FeatureWindowing               P:include/ksvm/windowing.hpp:13-21
AnovaKernelSpec                P:include/ksvm/kernel.hpp:17-19
Dataset                        P:include/ksvm/dataset.hpp:26-35 (points only)
KernelOperator                 P:include/ksvm/kernel.hpp:32-38
FastsumPlan / plan_fastsum     P:include/ksvm/fastsum.hpp:25-62
apply_fastsum                  P:include/ksvm/fastsum.hpp:65
apply_fastsum_cross            P:include/ksvm/fastsum.hpp:70-72
DomainError                    P:include/ksvm/fastsum.hpp:74-77
anova_fast_operator            P:include/ksvm/fastsum.hpp:81-84
=============================  =================================================

Exceptions: ``std::invalid_argument`` -> ``ValueError``; ``DomainError`` ->
:class:`DomainError`; CUDA/internal failures -> ``RuntimeError``.

Vectors may be numpy arrays (host: the call copies in, runs on the GPU and
copies out) or CUDA ``torch`` tensors (device: the work is ordered on
torch's current stream and the result is a CUDA tensor).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib

try:  # torch is plumbing only (device tensors, streams); optional on host
    import torch
except Exception:  # pragma: no cover
    torch = None


class DomainError(RuntimeError):
    """A cross-apply target falls outside the scaled torus ball (P:src/fastsum.cpp:316-320)."""


def _raise(code: int) -> None:
    if code == _lib.OK:
        return
    msg = _lib.last_error()
    if code == _lib.ERR_CONFIG:
        raise ValueError(msg)
    if code == _lib.ERR_DATA:
        raise DomainError(msg)
    raise RuntimeError(msg)


@dataclass
class FastsumConfig:
    bandwidth: int = 32        # N, even, per dimension
    window_cutoff: int = 4     # m, spreading half-width
    oversampling: int = 2      # sigma, oversampled grid edge M = sigma * N
    torus_radius: float = 0.25  # r_T (code default)

    def _c(self) -> _lib.Config:
        return _lib.Config(int(self.bandwidth), int(self.window_cutoff), int(self.oversampling),
                           float(self.torus_radius))

    def validate(self) -> None:
        c = self._c()
        _raise(_lib.load().ksvm_nfft_config_validate(C.byref(c)))


@dataclass
class GaussianKernelSpec:
    length_scale: float = 1.0


@dataclass
class FeatureWindowing:
    windows: list = field(default_factory=list)
    weights: list = field(default_factory=list)
    length_scales: list = field(default_factory=list)
    mi_scores: list = field(default_factory=list)

    def num_windows(self) -> int:
        return len(self.windows)

    @staticmethod
    def explicit(windows: Sequence[Sequence[int]], length_scales=None) -> "FeatureWindowing":
        """eta = 1/P, ell = 1 (P:src/pipeline.cpp:236-242)."""
        P = len(windows)
        return FeatureWindowing([list(w) for w in windows], [1.0 / P] * P,
                                list(length_scales) if length_scales is not None else [1.0] * P, [])


@dataclass
class AnovaKernelSpec:
    windowing: FeatureWindowing = field(default_factory=FeatureWindowing)


@dataclass
class Dataset:
    points: np.ndarray                 # n x d, row per sample
    labels: Optional[np.ndarray] = None

    def n(self) -> int:
        return int(self.points.shape[0])

    def dim(self) -> int:
        return int(self.points.shape[1])


class KernelOperator:
    """Symmetric PSD operator seam (P:include/ksvm/kernel.hpp:32-38)."""

    def size(self) -> int:
        raise NotImplementedError

    def apply(self, v):
        raise NotImplementedError

    def entry(self, i: int, j: int) -> float:
        raise NotImplementedError


# ---- argument marshalling -------------------------------------------------

def _is_cuda_tensor(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _host_matrix(pts) -> np.ndarray:
    if torch is not None and isinstance(pts, torch.Tensor):
        pts = pts.detach().cpu().numpy()
    a = np.asarray(pts, dtype=np.float64)
    if a.ndim == 1:
        a = a[:, None]
    if a.ndim != 2:
        raise ValueError("points must be an n x d matrix")
    return np.ascontiguousarray(a)


class _Vec:
    """Resolve a vector argument to (pointer, ptr_kind, stream) plus output."""

    def __init__(self, v, n: int, device: int):
        self.cuda = _is_cuda_tensor(v)
        if self.cuda:
            if v.dtype != torch.float64:
                raise ValueError("vectors must be float64")
            if v.device.index != device:
                raise ValueError(f"vector is on cuda:{v.device.index}, plan on cuda:{device}")
            self.t = v.contiguous()
            if self.t.numel() != n:
                raise ValueError("vector length mismatch")
            self.ptr = C.c_void_p(self.t.data_ptr())
            self.kind = _lib.DEVICE
            self.stream = C.c_void_p(torch.cuda.current_stream(v.device).cuda_stream)
        else:
            if torch is not None and isinstance(v, torch.Tensor):
                v = v.detach().numpy()
            self.t = np.ascontiguousarray(np.asarray(v, dtype=np.float64).reshape(-1))
            if self.t.shape[0] != n:
                raise ValueError("vector length mismatch")
            self.ptr = C.c_void_p(self.t.ctypes.data)
            self.kind = _lib.HOST
            self.stream = C.c_void_p(0)

    def out(self, m: int):
        if self.cuda:
            o = torch.empty(m, dtype=torch.float64, device=self.t.device)
            return o, C.c_void_p(o.data_ptr())
        o = np.empty(m, dtype=np.float64)
        return o, C.c_void_p(o.ctypes.data)


# ---- single-window plan ---------------------------------------------------

class FastsumPlan:
    """Per-window plan on one GPU (P:include/ksvm/fastsum.hpp:25-55)."""

    def __init__(self, handle, n: int, d: int, device: int):
        self._h = handle
        self._free = _lib.load().ksvm_nfft_plan_free  # kept: module globals may be gone in __del__
        self._n, self._d, self.device = n, d, device

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    def num_sources(self) -> int:
        return self._n

    def dim(self) -> int:
        return self._d

    def scaled_length(self) -> float:
        return float(_lib.load().ksvm_nfft_plan_scaled_length(self._h))

    def coefficient_sum(self) -> float:
        return float(_lib.load().ksvm_nfft_plan_coefficient_sum(self._h))

    def scale_points(self, pts) -> np.ndarray:
        a = _host_matrix(pts)
        if a.shape[1] != self._d:
            raise ValueError("scale_points: dimension mismatch")
        out = np.empty_like(a)
        _raise(_lib.load().ksvm_nfft_plan_scale_points(self._h, C.c_void_p(a.ctypes.data), a.shape[0],
                                                        a.shape[1], _lib.ROW_MAJOR,
                                                        C.c_void_p(out.ctypes.data)))
        return out


def plan_fastsum(points, spec=None, cfg: Optional[FastsumConfig] = None, fit_fraction: float = 1.0,
                 device: int = 0) -> FastsumPlan:
    """plan_fastsum (P:src/fastsum.cpp:103-209) on cuda:`device`."""
    cfg = cfg or FastsumConfig()
    ell = spec.length_scale if isinstance(spec, GaussianKernelSpec) else (1.0 if spec is None else float(spec))
    a = _host_matrix(points)
    n, d = a.shape
    h = C.c_void_p()
    c = cfg._c()
    _raise(_lib.load().ksvm_nfft_plan_create(C.c_void_p(a.ctypes.data), n, d, max(d, 1), _lib.ROW_MAJOR,
                                             float(ell), C.byref(c), float(fit_fraction), int(device),
                                             C.byref(h)))
    return FastsumPlan(h, n, d, int(device))


def apply_fastsum(plan: FastsumPlan, v):
    """K v at the plan's nodes (P:src/fastsum.cpp:300-305)."""
    n = plan.num_sources()
    if (v.numel() if _is_cuda_tensor(v) else np.asarray(v).size) != n:
        raise ValueError("apply_fastsum: vector length mismatch")
    a = _Vec(v, n, plan.device)
    out, optr = a.out(n)
    _raise(_lib.load().ksvm_nfft_plan_apply(plan._h, a.ptr, optr, a.kind, a.stream))
    return out


def apply_fastsum_cross(plan: FastsumPlan, targets, v):
    """t x n cross-kernel times v (P:src/fastsum.cpp:307-322); targets are raw coordinates."""
    n = plan.num_sources()
    if (v.numel() if _is_cuda_tensor(v) else np.asarray(v).size) != n:
        raise ValueError("apply_fastsum_cross: vector length mismatch")
    t = _host_matrix(targets)
    if t.shape[1] != plan.dim():
        raise ValueError("apply_fastsum_cross: target dimension mismatch")
    a = _Vec(v, n, plan.device)
    out, optr = a.out(t.shape[0])
    _raise(_lib.load().ksvm_nfft_plan_apply_cross(plan._h, C.c_void_p(t.ctypes.data), t.shape[0],
                                                  t.shape[1], _lib.ROW_MAJOR, a.ptr, optr, a.kind,
                                                  a.stream))
    return out


# ---- ANOVA operator -------------------------------------------------------

class AnovaFastOperator(KernelOperator):
    """sum_l eta_l K~_l as a KernelOperator (P:src/fastsum.cpp:326-362).

    ``window_mask`` (list of bools, one per window) restricts the windows
    whose fast applies run here (multi-GPU window sharding, see
    :mod:`paper_2312_00538_b200.sharding`); ``apply`` then returns the partial
    sum over the owned windows. ``precision`` is "fp64" (default) or "fp32"
    (north_star's optional fp32 mode: the d = 3 windows spread and gather in
    fp32, <= 1e-5 relative l2 against the fp64 reference).
    """

    def __init__(self, data, spec: AnovaKernelSpec, cfg: Optional[FastsumConfig] = None,
                 fit_fraction: float = 1.0, device: int = 0, window_mask=None, precision: str = "fp64"):
        cfg = cfg or FastsumConfig()
        pts = data.points if hasattr(data, "points") else data
        a = _host_matrix(pts)
        n, d = a.shape
        w = spec.windowing
        P = w.num_windows()
        feats = (C.c_int * max(1, sum(len(x) for x in w.windows)))(*[int(f) for x in w.windows for f in x])
        sizes = (C.c_int * max(1, P))(*[len(x) for x in w.windows])
        if len(w.weights) != P or len(w.length_scales) != P:
            raise ValueError("weights/length_scales size mismatch")
        eta = (C.c_double * max(1, P))(*[float(x) for x in w.weights])
        ell = (C.c_double * max(1, P))(*[float(x) for x in w.length_scales])
        mask = None
        if window_mask is not None:
            if len(window_mask) != P:
                raise ValueError("window_mask must have one entry per window")
            mask = (C.c_int * P)(*[1 if x else 0 for x in window_mask])
        c = cfg._c()
        h = C.c_void_p()
        _raise(_lib.load().ksvm_nfft_op_create(C.c_void_p(a.ctypes.data), n, d, d, _lib.ROW_MAJOR, feats,
                                               sizes, P, eta, ell, C.byref(c), float(fit_fraction), mask,
                                               int(device), _precision(precision), C.byref(h)))
        self._h = h
        self.precision = precision
        self._free = _lib.load().ksvm_nfft_op_free  # kept: module globals may be gone in __del__
        self._apply_fn = _lib.load().ksvm_nfft_op_apply
        self._n = n
        self.device = int(device)
        self.num_windows = P
        self.window_mask = list(window_mask) if window_mask is not None else [True] * P

    def __del__(self):
        h, free = getattr(self, "_h", None), getattr(self, "_free", None)
        if h and free is not None:
            free(h)
            self._h = None

    def size(self) -> int:
        return self._n

    def apply(self, v, out=None):
        # fast path: contiguous float64 numpy vectors (the per-iteration call
        # of a host-driven solver) -- no wrapper objects, one ctypes call
        if (type(v) is np.ndarray and v.dtype == np.float64 and v.ndim == 1 and v.shape[0] == self._n
                and v.flags.c_contiguous and (out is None or (type(out) is np.ndarray and out.dtype == np.float64
                                                              and out.shape == v.shape and out.flags.c_contiguous))):
            if out is None:
                out = np.empty(self._n)
            rc = self._apply_fn(self._h, v.__array_interface__["data"][0], out.__array_interface__["data"][0],
                                _lib.HOST, None)
            if rc:
                _raise(rc)
            return out
        a = _Vec(v, self._n, self.device)
        if out is None:
            out, optr = a.out(self._n)
        else:
            optr = C.c_void_p(out.data_ptr() if (torch is not None and isinstance(out, torch.Tensor))
                             else out.ctypes.data)
        _raise(_lib.load().ksvm_nfft_op_apply(self._h, a.ptr, optr, a.kind, a.stream))
        return out

    def apply_into(self, v, out) -> None:
        """Device-resident apply into a preallocated CUDA tensor (no allocation)."""
        if not (_is_cuda_tensor(v) and _is_cuda_tensor(out)):
            raise ValueError("apply_into takes CUDA tensors")
        st = C.c_void_p(torch.cuda.current_stream(v.device).cuda_stream)
        _raise(_lib.load().ksvm_nfft_op_apply(self._h, C.c_void_p(v.data_ptr()), C.c_void_p(out.data_ptr()),
                                              _lib.DEVICE, st))

    def apply_windows(self, v) -> None:
        """First half of the pipelined window-sharded matvec: every owned
        window's transform into its per-window output (CUDA tensor v)."""
        if not _is_cuda_tensor(v):
            raise ValueError("apply_windows takes a CUDA tensor")
        st = C.c_void_p(torch.cuda.current_stream(v.device).cuda_stream)
        _raise(_lib.load().ksvm_nfft_op_apply_windows(self._h, C.c_void_p(v.data_ptr()), _lib.DEVICE, st))

    def combine_range(self, y, lo: int, hi: int) -> None:
        """y[lo:hi] = sum_l eta_l out_l[lo:hi] over the owned windows (after
        apply_windows); equal to apply's rows bit for bit."""
        if not _is_cuda_tensor(y):
            raise ValueError("combine_range takes a CUDA tensor")
        st = C.c_void_p(torch.cuda.current_stream(y.device).cuda_stream)
        _raise(_lib.load().ksvm_nfft_op_combine_range(self._h, C.c_void_p(y.data_ptr()), int(lo), int(hi),
                                                      _lib.DEVICE, st))

    def apply_batch(self, V):
        """Y = K V for an n x k block (Nystrom sketch, P:src/low_rank.cpp:139-150)."""
        if _is_cuda_tensor(V):
            Vt = V.t().contiguous()  # k x n: column c at offset c*n
            Y = torch.empty_like(Vt)
            st = C.c_void_p(torch.cuda.current_stream(V.device).cuda_stream)
            _raise(_lib.load().ksvm_nfft_op_apply_batch(self._h, C.c_void_p(Vt.data_ptr()), C.c_void_p(Y.data_ptr()),
                                                        Vt.shape[0], self._n, _lib.DEVICE, st))
            return Y.t()
        Vt = np.ascontiguousarray(np.asarray(V, dtype=np.float64).T)
        Y = np.empty_like(Vt)
        _raise(_lib.load().ksvm_nfft_op_apply_batch(self._h, C.c_void_p(Vt.ctypes.data), C.c_void_p(Y.ctypes.data),
                                                    Vt.shape[0], self._n, _lib.HOST, C.c_void_p(0)))
        return Y.T

    def entry(self, i: int, j: int) -> float:
        return float(_lib.load().ksvm_nfft_op_entry(self._h, int(i), int(j)))

    def kernel_rows(self, rows, window: int = -1, device_out: bool = False):
        """Exact kernel rows K[rows, :] (window = -1: ANOVA; else one window's Gaussian)."""
        r = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1))
        rp = r.ctypes.data_as(C.POINTER(C.c_int64))
        if device_out:
            out = torch.empty((r.size, self._n), dtype=torch.float64, device=f"cuda:{self.device}")
            st = C.c_void_p(torch.cuda.current_stream(out.device).cuda_stream)
            _raise(_lib.load().ksvm_nfft_kernel_rows(self._h, int(window), rp, r.size, C.c_void_p(out.data_ptr()),
                                                     _lib.DEVICE, st))
            return out
        out = np.empty((r.size, self._n), dtype=np.float64)
        _raise(_lib.load().ksvm_nfft_kernel_rows(self._h, int(window), rp, r.size, C.c_void_p(out.ctypes.data),
                                                 _lib.HOST, C.c_void_p(0)))
        return out

    def kernel_diag(self, window: int = -1) -> np.ndarray:
        out = np.empty(self._n, dtype=np.float64)
        _raise(_lib.load().ksvm_nfft_kernel_diag(self._h, int(window), C.c_void_p(out.ctypes.data), _lib.HOST,
                                                 C.c_void_p(0)))
        return out

    def window_points(self, window: int) -> int:
        """Points the window is evaluated on (distinct points after the exact
        duplicate merge; 0 outside window_mask)."""
        return int(_lib.load().ksvm_nfft_op_window_points(self._h, int(window)))

    def set_stage_timing(self, on=True) -> None:
        """Record CUDA events between the launches of every apply: True / 1
        times every launch (dimension classes serialised), 2 times the main
        branch only (classes stay concurrent, as in an untimed apply)."""
        mode = 2 if on == 2 else (1 if on else 0)
        _raise(_lib.load().ksvm_nfft_op_set_stage_timing(self._h, mode))

    def last_stage_ms(self) -> dict:
        """{launch name: device ms} for each kernel launch of the last apply."""
        buf = (C.c_float * 24)()
        L = _lib.load()
        k = L.ksvm_nfft_op_last_stage_ms(self._h, buf, 24)
        out = {}
        for i in range(k):
            name = L.ksvm_nfft_op_stage_name(self._h, i).decode()
            out[name] = out.get(name, 0.0) + float(buf[i])
        return out


def _precision(p: str) -> int:
    table = {"fp64": _lib.FP64, "fp32": _lib.FP32}
    if p not in table:
        raise ValueError("precision must be 'fp64' or 'fp32'")
    return table[p]


def anova_fast_operator(data, spec: AnovaKernelSpec, cfg: Optional[FastsumConfig] = None,
                        fit_fraction: float = 1.0, device: int = 0, window_mask=None,
                        precision: str = "fp64") -> AnovaFastOperator:
    """anova_fast_operator (P:src/fastsum.cpp:366-371) on cuda:`device`."""
    return AnovaFastOperator(data, spec, cfg, fit_fraction, device, window_mask, precision)


# ---- prediction -------------------------------------------

def decision_values(train, spec: AnovaKernelSpec, coeff, bias: float, test, backend: str = "fast",
                    cfg: FastsumConfig = None, device: int = 0):
    """TrainedModel::decision_values (P:src/ipm.cpp:213-288) on the GPU:
    f = K(test, train) coeff + bias with coeff = alpha .* y; backend "fast"
    (per-window cross transforms, exact fallback outside the torus ball) or
    "exact". Points must already be normalized like the model's training
    data. Returns (f, number of targets evaluated exactly)."""
    tr = _host_matrix(train)
    te = _host_matrix(test)
    n, d = tr.shape
    if te.shape[1] != d:
        raise ValueError("predict: feature dimension mismatch")  # P:src/ipm.cpp:215-216
    w = spec.windowing
    feats = (C.c_int * max(1, sum(len(x) for x in w.windows)))(*[f for x in w.windows for f in x])
    sizes = (C.c_int * len(w.windows))(*[len(x) for x in w.windows])
    eta = np.ascontiguousarray(w.weights, dtype=np.float64)
    ell = np.ascontiguousarray(w.length_scales, dtype=np.float64)
    co = np.ascontiguousarray(np.asarray(coeff, dtype=np.float64).reshape(-1))
    if co.shape[0] != n:
        raise ValueError("coeff length mismatch")
    t = te.shape[0]
    out = np.empty(t)
    nex = C.c_int64(0)
    c = (cfg or FastsumConfig())._c()
    kind = {"fast": _lib.PREDICT_FAST, "exact": _lib.PREDICT_EXACT}[backend]
    _raise(_lib.load().ksvm_nfft_decision_values(C.c_void_p(tr.ctypes.data), n, d, d, _lib.ROW_MAJOR, feats, sizes,
                                                 len(w.windows), C.c_void_p(eta.ctypes.data),
                                                 C.c_void_p(ell.ctypes.data), C.byref(c), C.c_void_p(co.ctypes.data),
                                                 float(bias), C.c_void_p(te.ctypes.data), t, d, kind, int(device),
                                                 C.c_void_p(out.ctypes.data), C.byref(nex)))
    return out, int(nex.value)
