"""GPU parity: the B200 path vs the CPU oracle on identical seeded inputs.

Bar (north_star): relative l2 <= 1e-10 in fp64 against the reference's own
NFFT matvec (the oracle restatement, pinned bit-for-bit to the reference
compiled by path in tests/test_oracle.py). Inputs follow the reference's
tests (P:tests/test_fastsum.cpp, P:tests/helpers.hpp) and the BASELINE
configs (paper_2312_00538_b200/workloads.py).
"""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, DomainError, FastsumConfig,
                                   FeatureWindowing, GaussianKernelSpec, anova_fast_operator,
                                   apply_fastsum, apply_fastsum_cross, plan_fastsum)
from paper_2312_00538_b200 import workloads

pytestmark = pytest.mark.gpu

TOL = 1e-10  # relative l2, fp64 (BASELINE.json north_star)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def spec_of(windows, weights=None, ells=None):
    P = len(windows)
    return AnovaKernelSpec(FeatureWindowing([list(w) for w in windows],
                                            list(weights) if weights is not None else [1.0 / P] * P,
                                            list(ells) if ells is not None else [1.0] * P))


@pytest.mark.parametrize("d", [1, 2, 3])
def test_plan_apply_matches_oracle(oracle_lib, d):
    pts = oracle.random_points(500, d, 31)
    v = oracle.random_vector(500, 32)
    gp = plan_fastsum(pts, GaussianKernelSpec(1.0))
    op = oracle_lib.plan(pts)
    assert rel(apply_fastsum(gp, v), op.apply(v)) <= TOL
    assert gp.scaled_length() == pytest.approx(op.scaled_length(), rel=1e-15)
    assert gp.coefficient_sum() == pytest.approx(op.coefficient_sum(), rel=1e-12)


def test_anova_operator_matches_oracle(oracle_lib):
    # P:tests/test_fastsum.cpp:147-161 inputs
    pts = oracle.random_points(1000, 6, 61)
    v = oracle.random_vector(1000, 62)
    wins, eta, ell = [[0, 1, 2], [3, 4, 5]], [0.5, 0.5], [1.0, 1.3]
    g = anova_fast_operator(Dataset(pts), spec_of(wins, eta, ell))
    o = oracle_lib.anova(pts, wins, eta, ell)
    assert rel(g.apply(v), o.apply(v)) <= TOL
    assert g.entry(3, 8) == pytest.approx(o.entry(3, 8), rel=1e-14)


@pytest.mark.parametrize("cfg", [1, 2])
def test_baseline_config_matches_oracle(oracle_lib, cfg):
    w = workloads.make(cfg)
    g = anova_fast_operator(Dataset(w.points), spec_of(w.windows), fit_fraction=w.fit_fraction)
    o = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction)
    assert rel(g.apply(w.v), o.apply(w.v)) <= TOL


def test_bit_identical_reuse():
    # P:tests/test_fastsum.cpp:208-215
    pts = oracle.random_points(200, 2, 81)
    v = oracle.random_vector(200, 82)
    p = plan_fastsum(pts, GaussianKernelSpec(1.0))
    a, b = apply_fastsum(p, v), apply_fastsum(p, v)
    assert np.array_equal(a, b)
    w = workloads.config2(n=20000)
    op = anova_fast_operator(Dataset(w.points), spec_of(w.windows))
    assert np.array_equal(op.apply(w.v), op.apply(w.v))


def test_cross_apply_matches_oracle(oracle_lib):
    # P:tests/test_fastsum.cpp:108-145
    pts = oracle.random_points(300, 2, 51)
    v = oracle.random_vector(300, 52)
    gp, op = plan_fastsum(pts, 1.0), oracle_lib.plan(pts)
    tg = oracle.random_points(100, 2, 53, 0.5)
    assert rel(apply_fastsum_cross(gp, tg, v), op.apply_cross(tg, v)) <= TOL
    self_ = apply_fastsum(gp, v)
    cross = apply_fastsum_cross(gp, pts, v)
    assert np.abs(self_ - cross).max() <= 1e-12
    with pytest.raises(DomainError):
        apply_fastsum_cross(gp, np.array([[1e3, 1e3]]), v)


@pytest.mark.parametrize("N,m,sigma", [(8, 4, 2), (16, 4, 2), (32, 2, 2), (32, 3, 2), (32, 6, 2),
                                       (16, 8, 2), (32, 4, 1), (24, 4, 3)])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_other_parameters_match_oracle(oracle_lib, N, m, sigma, d):
    pts = oracle.random_points(400, d, 71)
    v = oracle.random_vector(400, 72)
    cfg = FastsumConfig(N, m, sigma, 0.25)
    gp = plan_fastsum(pts, 1.0, cfg)
    op = oracle_lib.plan(pts, 1.0, N, m, sigma, 0.25)
    assert rel(apply_fastsum(gp, v), op.apply(v)) <= TOL


def test_kernel_rows_and_diag():
    w = workloads.config1()
    op = anova_fast_operator(Dataset(w.points), spec_of(w.windows))
    rows = [0, 5, 1999]
    R = op.kernel_rows(rows, window=-1)
    x = w.points
    ref = np.zeros((3, w.n))
    for l, win in enumerate(w.windows):
        d2 = ((x[rows][:, None, win] - x[None, :, win]) ** 2).sum(-1)
        ref += 0.5 * np.exp(-d2)
    assert np.abs(R - ref).max() <= 1e-14
    R1 = op.kernel_rows(rows, window=1)
    d2 = ((x[rows][:, None, [3, 4, 5]] - x[None, :, [3, 4, 5]]) ** 2).sum(-1)
    assert np.abs(R1 - np.exp(-d2)).max() <= 1e-14
    assert np.all(op.kernel_diag(0) == 1.0)


@pytest.mark.parametrize("spread,gather", [("cell", "column"), ("column", "cell")])
@pytest.mark.parametrize("n,seed", [(3000, 91), (60000, 92)])
def test_d3_kernel_variants_match_oracle(oracle_lib, monkeypatch, spread, gather, n, seed):
    # both d = 3 spread and gather kernels (per-cell and column-blocked; the
    # engine picks by the mean points per cell) at sparse and dense cells,
    # for the operator and for a cross apply
    monkeypatch.setenv("KSVM_NFFT_SPREAD3", spread)
    monkeypatch.setenv("KSVM_NFFT_GATHER3", gather)
    pts = oracle.random_points(n, 3, seed)
    v = oracle.random_vector(n, seed + 1)
    g = anova_fast_operator(Dataset(pts), spec_of([[0, 1, 2]]))
    o = oracle_lib.anova(pts, [[0, 1, 2]])
    assert rel(g.apply(v), o.apply(v)) <= TOL
    p, q = plan_fastsum(pts, GaussianKernelSpec(1.0)), oracle_lib.plan(pts)
    tg = pts[: n // 3] * 0.9
    assert rel(apply_fastsum_cross(p, tg, v), q.apply_cross(tg, v)) <= TOL


def test_item_order_does_not_change_a_bit(monkeypatch):
    # items are dispatched largest first (KSVM_NFFT_LPT, default 1); patch
    # offsets travel with the items and every reduction keeps its plan order,
    # so the result is bit-identical to the (window, tile) order -- dense and
    # sparse d = 3 classes (cell / column kernels, column bounds permuted
    # with the items), d = 2 and d = 1 windows, heavy tiles split into items
    rng = np.random.default_rng(97)
    n = 120000
    x = np.concatenate([rng.normal(size=(n, 4)) * 0.3, rng.uniform(-1, 1, size=(n, 5))], axis=1)
    v = rng.normal(size=n)
    wins = [[0, 1, 2], [4, 5, 6], [3, 7], [8]]
    out = {}
    for order in ("0", "1", "2"):
        monkeypatch.setenv("KSVM_NFFT_LPT", order)
        out[order] = anova_fast_operator(Dataset(x), spec_of(wins)).apply(v)
    assert np.array_equal(out["0"], out["1"]) and np.array_equal(out["0"], out["2"])


@pytest.mark.parametrize("dedup", ["1", "0"])
def test_duplicate_points_match_oracle(oracle_lib, monkeypatch, dedup):
    # config-4-like windows: all-binary features (8 distinct points: the
    # exact-duplicate path), one mixed window and one continuous window
    monkeypatch.setenv("KSVM_NFFT_DEDUP", dedup)
    rng = np.random.default_rng(41)
    n = 20000
    X = np.empty((n, 9))
    X[:, 0:3] = rng.standard_normal((n, 3))
    X[:, 3] = rng.standard_normal(n)
    X[:, 4:9] = (rng.random((n, 5)) < 0.1).astype(float)
    X = (X - X.min(0)) / (X.max(0) - X.min(0)) * 0.5 - 0.25
    v = rng.standard_normal(n)
    wins = [[0, 1, 2], [3, 4, 5], [6, 7, 8]]
    g = anova_fast_operator(Dataset(X), spec_of(wins))
    o = oracle_lib.anova(X, wins)
    y = g.apply(v)
    assert rel(y, o.apply(v)) <= TOL
    assert np.array_equal(y, g.apply(v))
    # a 2-d and a 1-d binary window
    wins = [[4, 5], [6], [0, 1, 2]]
    g = anova_fast_operator(Dataset(X), spec_of(wins))
    assert rel(g.apply(v), oracle_lib.anova(X, wins).apply(v)) <= TOL
    # 4-level features: 64 distinct points per window (member-list sums),
    # next to register-bin and plain windows
    L = np.floor(rng.random((n, 3)) * 4) / 3 * 0.5 - 0.25
    X2 = np.hstack([X, L])
    wins = [[4, 5, 6], [9, 10, 11], [0, 1, 2], [7, 8]]
    g = anova_fast_operator(Dataset(X2), spec_of(wins))
    o = oracle_lib.anova(X2, wins)
    assert rel(g.apply(v), o.apply(v)) <= TOL
    V = rng.standard_normal((n, 3))
    Y = g.apply_batch(V)
    for c in range(3):
        assert rel(Y[:, c], o.apply(V[:, c])) <= TOL


def test_duplicate_config4_shape_matches_oracle(oracle_lib):
    w = workloads.make(4, 8000)
    g = anova_fast_operator(Dataset(w.points), spec_of(w.windows), fit_fraction=w.fit_fraction)
    o = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction)
    assert rel(g.apply(w.v), o.apply(w.v)) <= TOL


@pytest.mark.parametrize("grid", ["fused", "fused12", "conv3", "staged"])
@pytest.mark.parametrize("cfg,n,m", [(2, 60000, 4), (3, 8000, 4), (1, 2000, 4), (2, 5000, 3), (2, 4000, 6)])
def test_grid_side_variants_match_oracle(oracle_lib, monkeypatch, grid, cfg, n, m):
    # the fused grid side (reduce + separable convolution in one launch: a
    # thread-block cluster per 3-d window, one CTA per 1-/2-d window) and the
    # staged kernels, on operator data-range grids, m = 3 / 4 / 6
    monkeypatch.setenv("KSVM_NFFT_GRID", grid)
    w = workloads.make(cfg, n)
    c = FastsumConfig(window_cutoff=m)
    g = anova_fast_operator(Dataset(w.points), spec_of(w.windows), c, fit_fraction=w.fit_fraction)
    o = oracle_lib.anova(w.points, w.windows, m=m, fit=w.fit_fraction)
    y = g.apply(w.v)
    assert rel(y, o.apply(w.v)) <= TOL
    assert np.array_equal(y, g.apply(w.v))
