"""ORACLE / TEST INFRASTRUCTURE ONLY — CPU checkers for the B200 path.

Loads, via ctypes, the two CPU implementations that share the C ABI in
``oracle/ksvm_oracle.h``:

* ``Lib("oracle")`` - ``oracle/liboracle.so``, the Eigen-free restatement of
  the reference hot path (P:src/fastsum.cpp:103-371).
* ``Lib("ref")``    - ``oracle/_ref/libref.so``, the reference's own
  ``fastsum.cpp``/``kernel.cpp``/``windowing.cpp`` compiled unmodified by
  path (present when it was built in a container that has /root/reference;
  the built file travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_PATHS = {"oracle": os.path.join(HERE, "liboracle.so"),
          "ref": os.path.join(HERE, "_ref", "libref.so")}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref/libref.so when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def available(kind: str) -> bool:
    return os.path.exists(_PATHS[kind])


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Lib:
    """One of the two CPU libraries, with numpy-facing wrappers."""

    _cache: dict = {}

    def __init__(self, kind: str = "oracle"):
        if kind not in _PATHS:
            raise ValueError(kind)
        if not os.path.exists(_PATHS[kind]):
            raise FileNotFoundError(_PATHS[kind] + " (run oracle.build())")
        if kind not in Lib._cache:
            Lib._cache[kind] = self._bind(C.CDLL(_PATHS[kind]), kind)
        self.L = Lib._cache[kind]
        self.kind = kind
        self.p = kind + "_"

    @staticmethod
    def _bind(L, kind):
        p = kind + "_"
        vp = C.c_void_p
        sig = {
            "last_error": (C.c_char_p, []),
            "plan_create": (C.c_int, [_dp, C.c_int64, C.c_int, C.c_double, C.c_int, C.c_int,
                                      C.c_int, C.c_double, C.c_double, C.POINTER(vp)]),
            "plan_apply": (C.c_int, [vp, _dp, _dp]),
            "plan_apply_cross": (C.c_int, [vp, _dp, C.c_int64, _dp, _dp]),
            "plan_scaled_length": (C.c_double, [vp]),
            "plan_coefficient_sum": (C.c_double, [vp]),
            "plan_scale_points": (C.c_int, [vp, _dp, C.c_int64, _dp]),
            "plan_free": (None, [vp]),
            "anova_create": (C.c_int, [_dp, C.c_int64, C.c_int, _ip, _ip, C.c_int, _dp, _dp,
                                       C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.POINTER(vp)]),
            "anova_apply": (C.c_int, [vp, _dp, _dp]),
            "anova_entry": (C.c_double, [vp, C.c_int64, C.c_int64]),
            "anova_free": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, p + name)
            f.restype = res
            f.argtypes = args
        if kind == "oracle":
            for name, args in {"random_points": [C.c_int64, C.c_int64, C.c_uint64, C.c_double, _dp],
                               "random_vector": [C.c_int64, C.c_uint64, _dp],
                               "uniform": [C.c_int64, C.c_uint64, C.c_double, C.c_double, _dp],
                               "bernoulli": [C.c_int64, C.c_uint64, C.c_double, _dp],
                               "fft": [_dp, _dp, C.c_int, _ip, C.c_int]}.items():
                f = getattr(L, "oracle_" + name)
                f.restype = None
                f.argtypes = args
        return L

    def _fn(self, name):
        return getattr(self.L, self.p + name)

    def _check(self, code):
        if code != 0:
            raise OracleError(code, self._fn("last_error")().decode())

    # --- per-window plan (P:include/ksvm/fastsum.hpp:25-72) -------------
    def plan(self, pts, ell=1.0, N=32, m=4, sigma=2, torus_radius=0.25, fit=1.0):
        return Plan(self, pts, ell, N, m, sigma, torus_radius, fit)

    # --- ANOVA operator (P:src/fastsum.cpp:326-371) -----------------------
    def anova(self, pts, windows, weights=None, ells=None, N=32, m=4, sigma=2,
              torus_radius=0.25, fit=1.0):
        return Anova(self, pts, windows, weights, ells, N, m, sigma, torus_radius, fit)


class Plan:
    def __init__(self, lib, pts, ell, N, m, sigma, rT, fit):
        pts = np.asarray(pts, dtype=np.float64)
        if pts.ndim == 1:
            pts = pts[:, None]
        self.lib, self.n, self.d = lib, pts.shape[0], pts.shape[1]
        cm = _f64(pts.T)  # column-major n x d
        h = C.c_void_p()
        lib._check(lib._fn("plan_create")(_ptr(cm), self.n, self.d, ell, N, m, sigma, rT, fit,
                                          C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib._fn("plan_free")(self.h)
            self.h = None

    def apply(self, v):
        v = _f64(v)
        out = np.empty(self.n)
        self.lib._check(self.lib._fn("plan_apply")(self.h, _ptr(v), _ptr(out)))
        return out

    def apply_cross(self, targets, v):
        t = np.asarray(targets, dtype=np.float64)
        if t.ndim == 1:
            t = t[:, None]
        cm = _f64(t.T)
        v = _f64(v)
        out = np.empty(t.shape[0])
        self.lib._check(self.lib._fn("plan_apply_cross")(self.h, _ptr(cm), t.shape[0], _ptr(v),
                                                         _ptr(out)))
        return out

    def scaled_length(self):
        return self.lib._fn("plan_scaled_length")(self.h)

    def coefficient_sum(self):
        return self.lib._fn("plan_coefficient_sum")(self.h)

    def scale_points(self, pts):
        t = np.asarray(pts, dtype=np.float64)
        if t.ndim == 1:
            t = t[:, None]
        cm = _f64(t.T)
        out = np.empty_like(cm)
        self.lib._check(self.lib._fn("plan_scale_points")(self.h, _ptr(cm), t.shape[0], _ptr(out)))
        return out.T.copy()


class Anova:
    def __init__(self, lib, pts, windows, weights, ells, N, m, sigma, rT, fit):
        pts = _f64(pts)
        self.lib, self.n = lib, pts.shape[0]
        P = len(windows)
        feats = np.ascontiguousarray([f for w in windows for f in w], dtype=np.int32)
        sizes = np.ascontiguousarray([len(w) for w in windows], dtype=np.int32)
        weights = _f64(weights if weights is not None else [1.0 / P] * P)
        ells = _f64(ells if ells is not None else [1.0] * P)
        h = C.c_void_p()
        lib._check(lib._fn("anova_create")(_ptr(pts), self.n, pts.shape[1],
                                           feats.ctypes.data_as(_ip), sizes.ctypes.data_as(_ip),
                                           P, _ptr(weights), _ptr(ells), N, m, sigma, rT, fit,
                                           C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib._fn("anova_free")(self.h)
            self.h = None

    def apply(self, v):
        v = _f64(v)
        out = np.empty(self.n)
        self.lib._check(self.lib._fn("anova_apply")(self.h, _ptr(v), _ptr(out)))
        return out

    def entry(self, i, j):
        return self.lib._fn("anova_entry")(self.h, i, j)


# --- input generators (P:tests/helpers.hpp:15-31) --------------------------
def random_points(n, d, seed, scale=1.0) -> np.ndarray:
    """n x d (row-major numpy) drawn exactly like helpers::random_points."""
    L = Lib("oracle").L
    out = np.empty(n * d)
    L.oracle_random_points(n, d, seed, scale, _ptr(out))
    return out.reshape(d, n).T.copy()


def random_vector(n, seed) -> np.ndarray:
    L = Lib("oracle").L
    out = np.empty(n)
    L.oracle_random_vector(n, seed, _ptr(out))
    return out


def uniform(n, seed, lo, hi) -> np.ndarray:
    L = Lib("oracle").L
    out = np.empty(n)
    L.oracle_uniform(n, seed, lo, hi, _ptr(out))
    return out


def bernoulli(n, seed, p) -> np.ndarray:
    L = Lib("oracle").L
    out = np.empty(n)
    L.oracle_bernoulli(n, seed, p, _ptr(out))
    return out


def fft(x: np.ndarray, sign: int = -1) -> np.ndarray:
    """Unnormalised multi-dimensional DFT of the oracle (FFTW sign convention)."""
    L = Lib("oracle").L
    a = np.ascontiguousarray(x, dtype=np.complex128)
    out = np.empty_like(a)
    dims = np.ascontiguousarray(a.shape, dtype=np.int32)
    L.oracle_fft(a.ctypes.data_as(_dp), out.ctypes.data_as(_dp), a.ndim, dims.ctypes.data_as(_ip), sign)
    return out


def dense_gaussian(pts, ell=1.0) -> np.ndarray:
    """helpers::dense_gaussian (P:tests/helpers.hpp:78-89)."""
    pts = np.asarray(pts, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts[:, None]
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    return np.exp(-d2 / (ell * ell))


# --- Newton saddle system (oracle/saddle_oracle.cpp, P:src/saddle.cpp) ------
def _saddle_lib():
    L = Lib("oracle").L
    if not getattr(L, "_saddle_bound", False):
        vp = C.c_void_p
        L.oracle_saddle_last_error.restype = C.c_char_p
        L.oracle_saddle_apply.restype = C.c_int
        L.oracle_saddle_apply.argtypes = [vp, vp, C.c_int64, _dp, _dp, _dp, _dp]
        L.oracle_precond_apply.restype = C.c_int
        L.oracle_precond_apply.argtypes = [vp, C.c_int, C.c_int64, _dp, _dp, _dp, _dp, _ip]
        L.oracle_gmres_solve.restype = C.c_int
        L.oracle_gmres_solve.argtypes = [vp, vp, C.c_int64, _dp, _dp, vp, C.c_int, _dp, C.c_double, C.c_int,
                                         _dp, _dp, _dp]
        L._saddle_bound = True
    return L


def _saddle_check(L, code):
    if code != 0:
        raise OracleError(code, L.oracle_saddle_last_error().decode())


def _kop(K):
    """K: an oracle Anova (the NFFT operator) or a dense n x n matrix."""
    if isinstance(K, Anova):
        return K.h, None, K.n, None
    D = np.ascontiguousarray(K, dtype=np.float64)
    return None, C.c_void_p(D.ctypes.data), D.shape[0], D


def saddle_apply(K, y, theta, vw) -> np.ndarray:
    """SaddleOperator::apply (P:src/saddle.cpp:22-33)."""
    L = _saddle_lib()
    h, dense, n, keep = _kop(K)
    y, theta, vw = _f64(y), _f64(theta), _f64(vw)
    out = np.empty(n + 1)
    _saddle_check(L, L.oracle_saddle_apply(h, dense, n, _ptr(y), _ptr(theta), _ptr(vw), _ptr(out)))
    return out


def precond_apply(Z, y, theta, g):
    """SaddlePreconditioner(refresh(theta)).apply(g) (P:src/saddle.cpp:41-90);
    Z None -> identity. Returns (out, diagonal_fallback)."""
    L = _saddle_lib()
    y, theta, g = _f64(y), _f64(theta), _f64(g)
    n = y.shape[0]
    Zc = None if Z is None else np.ascontiguousarray(Z, dtype=np.float64)
    out = np.empty(n + 1)
    fb = C.c_int(0)
    _saddle_check(L, L.oracle_precond_apply(None if Zc is None else C.c_void_p(Zc.ctypes.data),
                                            0 if Zc is None else Zc.shape[0], n, _ptr(y), _ptr(theta), _ptr(g),
                                            _ptr(out), C.byref(fb)))
    return out, bool(fb.value)


def gmres_solve(K, y, theta, Z, rhs, tol, max_iter):
    """gmres_solve with SaddleOperator(K, y, theta) and
    SaddlePreconditioner(Z, y) refreshed at theta (P:src/saddle.cpp:92-178).
    Returns (x, stats dict with residual_history)."""
    L = _saddle_lib()
    h, dense, n, keep = _kop(K)
    y, theta, rhs = _f64(y), _f64(theta), _f64(rhs)
    Zc = None if Z is None else np.ascontiguousarray(Z, dtype=np.float64)
    x = np.empty(n + 1)
    st = np.zeros(4)
    hist = np.zeros(max(max_iter, 1))
    _saddle_check(L, L.oracle_gmres_solve(h, dense, n, _ptr(y), _ptr(theta),
                                          None if Zc is None else C.c_void_p(Zc.ctypes.data),
                                          0 if Zc is None else Zc.shape[0], _ptr(rhs), float(tol), int(max_iter),
                                          _ptr(x), _ptr(st), _ptr(hist)))
    it = int(st[0])
    return x, {"iterations": it, "relative_residual": float(st[1]), "converged": bool(st[2]),
               "breakdown": bool(st[3]), "residual_history": hist[:it].copy()}


# --- greedy pivoted Cholesky (oracle/lowrank_oracle.cpp, P:src/low_rank.cpp) --
def _lowrank_lib():
    L = Lib("oracle").L
    if not getattr(L, "_lowrank_bound", False):
        L.oracle_lowrank_last_error.restype = C.c_char_p
        L.oracle_pivoted_cholesky.restype = C.c_int
        L.oracle_pivoted_cholesky.argtypes = [_dp, C.c_int64, C.c_int, _ip, _ip, C.c_int, _dp, _dp, C.c_int,
                                              C.c_int, C.c_double, _dp, _ip, _dp, C.POINTER(C.c_int64)]
        L.oracle_pivoted_cholesky_dense.restype = C.c_int
        L.oracle_pivoted_cholesky_dense.argtypes = [_dp, C.c_int64, C.c_int, C.c_double, _dp, _ip, _dp,
                                                    C.POINTER(C.c_int64)]
        L._lowrank_bound = True
    return L


def pivoted_cholesky_dense(M, rank, err_tol=0.0):
    """pivoted_cholesky_greedy over a DenseOperator (P:tests/helpers.hpp).
    Returns (Z r x n, trace_residual, pivots)."""
    L = _lowrank_lib()
    M = np.ascontiguousarray(M, dtype=np.float64)
    n = M.shape[0]
    rr = max(1, min(int(rank), n))
    Z = np.zeros(rr * n)
    piv = np.zeros(rr, dtype=np.int64)
    r, tr = C.c_int(0), C.c_double(0.0)
    code = L.oracle_pivoted_cholesky_dense(_ptr(M), n, int(rank), float(err_tol), _ptr(Z), C.byref(r), C.byref(tr),
                                           piv.ctypes.data_as(C.POINTER(C.c_int64)))
    if code != 0:
        raise OracleError(code, L.oracle_lowrank_last_error().decode())
    return Z[: r.value * n].reshape(r.value, n), tr.value, piv[: r.value]


def pivoted_cholesky(pts, windows, window=0, rank=10, err_tol=0.0, weights=None, ells=None):
    """pivoted_cholesky_greedy over WindowOperator(window) (window >= 0) or
    the ANOVA entries (window = -1). Returns (Z r x n, trace_residual, pivots)."""
    L = _lowrank_lib()
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n, d = pts.shape
    P = len(windows)
    feats = np.ascontiguousarray([f for w in windows for f in w], dtype=np.int32)
    sizes = np.ascontiguousarray([len(w) for w in windows], dtype=np.int32)
    weights = _f64(weights if weights is not None else [1.0 / P] * P)
    ells = _f64(ells if ells is not None else [1.0] * P)
    rr = max(1, min(int(rank), n))
    Z = np.zeros(rr * n)
    piv = np.zeros(rr, dtype=np.int64)
    r = C.c_int(0)
    tr = C.c_double(0.0)
    code = L.oracle_pivoted_cholesky(_ptr(pts), n, d, feats.ctypes.data_as(_ip), sizes.ctypes.data_as(_ip), P,
                                     _ptr(weights), _ptr(ells), int(window), int(rank), float(err_tol), _ptr(Z),
                                     C.byref(r), C.byref(tr), piv.ctypes.data_as(C.POINTER(C.c_int64)))
    if code != 0:
        raise OracleError(code, L.oracle_lowrank_last_error().decode())
    return Z[: r.value * n].reshape(r.value, n), tr.value, piv[: r.value]


# --- prediction (P:src/ipm.cpp:213-288, TrainedModel::decision_values) -------
def decision_values(train, windows, weights, ells, coeff, bias, test, fast=True, N=32, m=4, sigma=2,
                    torus_radius=0.25, kind="oracle"):
    """Restatement of decision_values on the oracle's (or the reference
    build's, kind="ref") plans: kFast per-window cross transforms over
    targets with ||scaled|| <= r_T, exact sums for the rest; kExact all
    exact (anova_eval, P:src/kernel.cpp:15-29). Returns (f + bias, #exact)."""
    lib = Lib(kind)
    train = np.asarray(train, dtype=np.float64)
    test = np.asarray(test, dtype=np.float64)
    coeff = _f64(coeff)
    t = test.shape[0]
    f = np.zeros(t)
    offending = np.full(t, not fast)
    if fast:
        for l, win in enumerate(windows):
            plan = lib.plan(train[:, win], ells[l], N, m, sigma, torus_radius, 1.0 / 1.2)
            sc = plan.scale_points(test[:, win])
            ok = np.sqrt((sc * sc).sum(axis=1)) <= torus_radius
            offending |= ~ok
            if ok.any():
                part = plan.apply_cross(test[ok][:, win], coeff)
                f[np.nonzero(ok)[0]] += weights[l] * part
    redo = np.nonzero(offending)[0]
    for j in redo:  # exact_rows: acc += coeff_i * anova_eval(x_i, t_j)
        acc = 0.0
        x = test[j]
        for i in range(train.shape[0]):
            s = 0.0
            for l, win in enumerate(windows):
                d2 = 0.0
                for fidx in win:
                    diff = train[i, fidx] - x[fidx]
                    d2 += diff * diff
                s += weights[l] * np.exp(-d2 / (ells[l] * ells[l]))
            acc += coeff[i] * s
        f[j] = acc
    return f + bias, len(redo)


# --- interior point loop (P:src/ipm.cpp) --------------------------------------
IPM_DEFAULTS = {"C": 0.5, "sigma": 0.6, "gamma0": 0.99995, "tol_ip": 1e-1, "max_ip_iters": 50,
                "tol_gmres": 1e-3, "max_gmres_iters": 100, "mu0": 1.0}  # P:include/ksvm/ipm.hpp:15-24


def _ipm_lib():
    L = _saddle_lib()
    if not getattr(L, "_ipm_bound", False):
        vp = C.c_void_p
        L.oracle_ipm_train.restype = C.c_int
        L.oracle_ipm_train.argtypes = [vp, vp, C.c_int64, _dp, vp, C.c_int, _dp, _dp, _dp, vp]
        L.oracle_compute_bias.restype = C.c_int
        L.oracle_compute_bias.argtypes = [vp, vp, C.c_int64, _dp, _dp, C.c_double, C.c_double, _dp]
        L.oracle_blobs.restype = None
        L.oracle_blobs.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_uint64, C.c_double, _dp, _dp]
        L._ipm_bound = True
    return L


def ipm_train(K, y, Z=None, **cfg):
    """ipm_train (P:src/ipm.cpp:76-155). K: oracle Anova or dense matrix.
    Returns (alpha, result dict, per-iteration log array)."""
    L = _ipm_lib()
    c = dict(IPM_DEFAULTS, **cfg)
    carr = _f64([c[k] for k in ("C", "sigma", "gamma0", "tol_ip", "max_ip_iters", "tol_gmres", "max_gmres_iters",
                                 "mu0")])
    h, dense, n, keep = _kop(K)
    y = _f64(y)
    Zc = None if Z is None else np.ascontiguousarray(Z, dtype=np.float64)
    alpha = np.empty(n)
    res = np.zeros(7)
    log = np.zeros((int(c["max_ip_iters"]), 6))
    _saddle_check(L, L.oracle_ipm_train(h, dense, n, _ptr(y), None if Zc is None else C.c_void_p(Zc.ctypes.data),
                                        0 if Zc is None else Zc.shape[0], _ptr(carr), _ptr(alpha), _ptr(res),
                                        C.c_void_p(log.ctypes.data)))
    it = int(res[5])
    status = {0: "converged", 1: "max_iterations", 2: "stalled"}[int(res[4])]
    return alpha, {"lambda": res[0], "mu_final": res[1], "xi_alpha_rel": res[2], "xi_lambda_rel": res[3],
                   "status": status, "iterations": it, "mean_gmres_iters": res[6]}, log[:it].copy()


def compute_bias(K, alpha, y, C, eps_sv):
    """compute_bias (P:src/ipm.cpp:157-185)."""
    L = _ipm_lib()
    h, dense, n, keep = _kop(K)
    alpha, y = _f64(alpha), _f64(y)
    b = np.zeros(1)
    _saddle_check(L, L.oracle_compute_bias(h, dense, n, _ptr(alpha), _ptr(y), float(C), float(eps_sv), _ptr(b)))
    return float(b[0])


def blobs(n, d, gap, seed, noise=0.5):
    """helpers::blobs (P:tests/helpers.hpp:41-56): (n x d points, labels)."""
    L = _ipm_lib()
    pts = np.empty(n * d)
    lab = np.empty(n)
    L.oracle_blobs(n, d, gap, seed, noise, _ptr(pts), _ptr(lab))
    return pts.reshape(d, n).T.copy(), lab


# --- training-data preparation (P:src/dataset.cpp:212-282) -------------------
def balance_and_split(labels, train_fraction=0.5, seed=0, kind="oracle"):
    """balance_and_split as (train_idx sorted, test_idx) row indices; kind
    "ref" runs the reference's own dataset.cpp (oracle/_ref)."""
    L = Lib(kind).L
    f = getattr(L, kind + "_balance_and_split")
    lp = C.POINTER(C.c_int64)
    f.restype = C.c_int
    f.argtypes = [_dp, C.c_int64, C.c_double, C.c_uint64, lp, lp, lp, lp]
    lab = _f64(labels)
    n = lab.shape[0]
    tr = np.zeros(max(n, 1), dtype=np.int64)
    te = np.zeros(max(n, 1), dtype=np.int64)
    ntr, nte = C.c_int64(0), C.c_int64(0)
    code = f(_ptr(lab), n, float(train_fraction), int(seed), tr.ctypes.data_as(lp), C.byref(ntr),
             te.ctypes.data_as(lp), C.byref(nte))
    if code != 0:
        raise OracleError(code, "balance_and_split failed")
    return tr[: ntr.value].copy(), te[: nte.value].copy()


def zscore(train, test=None, kind="oracle"):
    """zscore_fit_transform: returns (train_z, test_z, means, stddevs)."""
    L = Lib(kind).L
    f = getattr(L, kind + "_zscore")
    f.restype = C.c_int
    f.argtypes = [_dp, C.c_int64, _dp, C.c_int64, C.c_int, _dp, _dp]
    tr = np.asfortranarray(np.asarray(train, dtype=np.float64))
    n, d = tr.shape
    te = None if test is None else np.asfortranarray(np.asarray(test, dtype=np.float64))
    nt = 0 if te is None else te.shape[0]
    mu, sd = np.zeros(d), np.zeros(d)
    code = f(tr.ctypes.data_as(_dp), n, None if te is None else te.ctypes.data_as(_dp), nt, d, _ptr(mu), _ptr(sd))
    if code != 0:
        raise OracleError(code, "zscore failed")
    return np.ascontiguousarray(tr), None if te is None else np.ascontiguousarray(te), mu, sd


# --- Nystrom factor (oracle/nystrom_oracle.cpp, P:src/low_rank.cpp:115-168) ---
NYSTROM_COLUMNS, NYSTROM_GAUSSIAN = 0, 1


def _nystrom_lib():
    L = Lib("oracle").L
    if not getattr(L, "_nystrom_bound", False):
        L.oracle_nystrom_last_error.restype = C.c_char_p
        L.oracle_nystrom_dense.restype = C.c_int
        L.oracle_nystrom_dense.argtypes = [_dp, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_double, _dp]
        L.oracle_nystrom_window.restype = C.c_int
        L.oracle_nystrom_window.argtypes = [_dp, C.c_int64, C.c_int, _ip, C.c_int, C.c_double, C.c_void_p, C.c_int,
                                            C.c_int, C.c_uint64, C.c_double, _dp]
        L._nystrom_bound = True
    return L


def nystrom_dense(M, rank, mode, seed, ldl_threshold=1e-8):
    """nystrom(DenseOperator(M), rank, mode, seed): Z (rank x n)."""
    L = _nystrom_lib()
    M = np.ascontiguousarray(M, dtype=np.float64)
    n = M.shape[0]
    Z = np.zeros(max(int(rank), 1) * n)
    code = L.oracle_nystrom_dense(_ptr(M), n, int(rank), int(mode), int(seed), float(ldl_threshold), _ptr(Z))
    if code != 0:
        raise OracleError(code, L.oracle_nystrom_last_error().decode())
    return Z.reshape(-1, n)[: int(rank)]


def nystrom_window(pts, feats, ell, rank, mode, seed, ldl_threshold=1e-8, N=32, m=4, sigma=2, torus_radius=0.25):
    """nystrom over one window of row-major points: mode 0 on the exact
    WindowOperator, mode 1 on the FastWindowOperator (plan fit 1.0,
    P:src/pipeline.cpp:114-133)."""
    L = _nystrom_lib()
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    n, d = pts.shape
    f = np.ascontiguousarray(feats, dtype=np.int32)
    plan = Lib("oracle").plan(pts[:, f], ell, N, m, sigma, torus_radius, 1.0) if mode == 1 else None
    Z = np.zeros(max(int(rank), 1) * n)
    code = L.oracle_nystrom_window(_ptr(pts), n, d, f.ctypes.data_as(_ip), len(f), float(ell),
                                   plan.h if plan is not None else None, int(rank), int(mode), int(seed),
                                   float(ldl_threshold), _ptr(Z))
    if code != 0:
        raise OracleError(code, L.oracle_nystrom_last_error().decode())
    return Z.reshape(-1, n)[: int(rank)]


# --- the reference's own host driver (oracle/driver, oracle/_ref/libdriver_*.so) ---
class Driver:
    """The reference's train_pipeline / gmres_solve compiled unmodified by path
    (P:src/{dataset,windowing,kernel,low_rank,saddle,ipm,pipeline}.cpp)
    against oracle/shim2, with either the reference's own fastsum.cpp
    (kind "cpu") or the drop-in paper_2312_00538_b200/cpp/ksvm_fastsum_gpu.cpp
    on libksvm_nfft.so (kind "gpu")."""

    PRECOND = {"none": 0, "cholesky-greedy": 1, "nystrom-gaussian": 4}

    def __init__(self, kind: str = "cpu"):
        path = os.path.join(HERE, "_ref", f"libdriver_{kind}.so")
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (built by `make -C oracle` where /root/reference exists)")
        self.L = C.CDLL(path)
        self.L.drv_last_error.restype = C.c_char_p
        self.L.drv_train_pipeline.restype = C.c_int
        self.L.drv_train_pipeline.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_char_p, C.c_int, C.c_int,
                                              C.c_double, C.c_uint64, C.c_int, _dp, _dp, _dp, _dp]
        self.L.drv_train_steps.restype = C.c_int
        self.L.drv_train_steps.argtypes = [_dp, _dp, C.c_int64, C.c_int, C.c_char_p, C.c_int, C.c_int, C.c_double,
                                           C.c_uint64, _dp, _dp, _dp, _dp, C.c_int]
        self.L.drv_gmres.restype = C.c_int
        self.L.drv_gmres.argtypes = [_dp, C.c_int64, C.c_int, C.c_char_p, _dp, _dp, _dp, C.c_int, _dp,
                                     C.c_double, C.c_int, _dp, _dp]

    @staticmethod
    def available(kind: str) -> bool:
        return os.path.exists(os.path.join(HERE, "_ref", f"libdriver_{kind}.so"))

    def _check(self, code):
        if code != 0:
            raise OracleError(code, self.L.drv_last_error().decode())

    def train_pipeline(self, points, labels, windows, precond="cholesky-greedy", rank=200, C_=1.0, seed=0,
                       fast=True):
        """ksvm::train_pipeline; returns a dict with the TrainReport fields, the
        dual objective, alpha, bias and the held-out split's decision values
        and labels."""
        X = _f64(points)
        n, d = X.shape
        lab = _f64(labels)
        spec = windows if isinstance(windows, str) else ";".join(",".join(str(f) for f in w) for w in windows)
        scal = np.zeros(12)
        alpha = np.zeros(n)
        dec = np.zeros(n)
        tl = np.zeros(n)
        self._check(self.L.drv_train_pipeline(_ptr(X), _ptr(lab), n, d, spec.encode(), self.PRECOND[precond],
                                              int(rank), float(C_), int(seed), 1 if fast else 0, _ptr(scal),
                                              _ptr(alpha), _ptr(dec), _ptr(tl)))
        ntr, nte = int(scal[0]), int(scal[1])
        return {"n_train": ntr, "n_test": nte, "ipm_iters": int(scal[2]), "mean_gmres": scal[3],
                "status": int(scal[4]), "rank": int(scal[5]), "xi_alpha": scal[6], "xi_lambda": scal[7],
                "mu_final": scal[8], "dual_objective": scal[9], "bias": scal[10], "dual_feasibility": scal[11],
                "alpha": alpha[:ntr].copy(), "test_decision": dec[:nte].copy(), "test_labels": tl[:nte].copy()}

    def train_steps(self, points, labels, windows, precond="cholesky-greedy", rank=200, C_=1.0, seed=0):
        """train_on_prepared's steps on the reference's functions (fast
        backend), with the per-Newton-step log: rows (mu, xi_alpha_rel,
        xi_lambda_rel, step_alpha, gmres_iterations, gmres_converged)."""
        X = _f64(points)
        n, d = X.shape
        spec = windows if isinstance(windows, str) else ";".join(",".join(str(f) for f in w) for w in windows)
        scal = np.zeros(12)
        alpha = np.zeros(n)
        dec = np.zeros(n)
        log = np.zeros(6 * 64)
        self._check(self.L.drv_train_steps(_ptr(X), _ptr(_f64(labels)), n, d, spec.encode(), self.PRECOND[precond],
                                           int(rank), float(C_), int(seed), _ptr(scal), _ptr(alpha), _ptr(dec),
                                           _ptr(log), 64))
        ntr, nte, its = int(scal[0]), int(scal[1]), int(scal[2])
        return {"n_train": ntr, "n_test": nte, "ipm_iters": its, "mean_gmres": scal[3], "status": int(scal[4]),
                "rank": int(scal[5]), "xi_alpha": scal[6], "xi_lambda": scal[7], "mu_final": scal[8],
                "dual_objective": scal[9], "bias": scal[10], "lambda": scal[11], "alpha": alpha[:ntr].copy(),
                "test_decision": dec[:nte].copy(), "log": log[:6 * its].reshape(its, 6).copy()}

    def gmres(self, points, windows, y, theta, Z, rhs, tol=1e-3, max_iter=100):
        """ksvm::gmres_solve on the fast operator (fit 1/1.2) with the
        reference's SaddlePreconditioner of the stacked factor Z (k x n)."""
        X = _f64(points)
        n, d = X.shape
        spec = windows if isinstance(windows, str) else ";".join(",".join(str(f) for f in w) for w in windows)
        k = 0 if Z is None else int(np.asarray(Z).shape[0])
        Zc = _f64(Z) if k else np.zeros(1)
        x = np.zeros(n + 1)
        scal = np.zeros(4)
        self._check(self.L.drv_gmres(_ptr(X), n, d, spec.encode(), _ptr(_f64(y)), _ptr(_f64(theta)), _ptr(Zc), k,
                                     _ptr(_f64(rhs)), float(tol), int(max_iter), _ptr(x), _ptr(scal)))
        return x, {"iterations": int(scal[0]), "relative_residual": scal[1], "converged": bool(scal[2]),
                   "diagonal_fallback": bool(scal[3])}
