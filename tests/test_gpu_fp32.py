"""GPU parity of the optional fp32 mode (BASELINE north_star: "<= 1e-5 in an
optional fp32 mode") against the fp64 reference fastsum.

The d = 3, m = 4 windows with dense cells spread and gather in fp32
(csrc/nfft_f32.cu: the 3xTF32 tensor-core kernels by default, the FFMA kernels
with KSVM_NFFT_F32K=ffma; both are tested); sparse-cell classes (configs 1, 2), the grid stage, the
d <= 2 windows and the window sum stay fp64. KSVM_NFFT_F32=all forces the
fp32 kernels on sparse cells too, so they are tested there as well. The checker is
the oracle restatement (bit-identical to the reference's own
P:src/fastsum.cpp, tests/test_oracle.py), at full size for BASELINE configs
1-3 and on seeded subsamples of configs 4 and 5 (the fp64 full-size runs are
tests/test_gpu_fullsize_parity.py). Bar: relative l2 <= 1e-5.
"""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FastsumConfig, FeatureWindowing, _lib,
                                   anova_fast_operator, workloads)

pytestmark = pytest.mark.gpu

TOL32 = 1e-5  # relative l2 (BASELINE.json north_star, optional fp32 mode)


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def spec_of(windows, ells=None):
    P = len(windows)
    return AnovaKernelSpec(FeatureWindowing([list(w) for w in windows], [1.0 / P] * P,
                                            list(ells) if ells is not None else [1.0] * P))


def fp32_op(w, **kw):
    return anova_fast_operator(Dataset(w.points), spec_of(w.windows), fit_fraction=w.fit_fraction,
                               precision="fp32", **kw)


@pytest.mark.parametrize("kernels", ["tf32", "ffma"])
@pytest.mark.parametrize("cfg,n", [(1, None), (2, None), (3, None), (4, 50000), (5, 200000)])
def test_fp32_matches_fp64_oracle(oracle_lib, monkeypatch, cfg, n, kernels):
    monkeypatch.setenv("KSVM_NFFT_F32", "all")  # fp32 kernels even on sparse cells
    monkeypatch.setenv("KSVM_NFFT_F32K", kernels)
    w = workloads.make(cfg, n)
    ref = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)
    before = _lib.launch_count()
    y = fp32_op(w).apply(w.v)
    assert _lib.launch_count() > before
    e = rel(y, ref)
    assert e <= TOL32, e
    # it really is the fp32 path: the fp64 path matches the oracle to ~1e-15
    assert e > 1e-10, e


@pytest.mark.parametrize("cfg,n", [(2, None), (5, 200000)])
def test_fp32_default_density_rule(oracle_lib, cfg, n):
    # default: sparse-cell classes (config 2) keep the exact fp64 kernels,
    # dense ones (config 5) run fp32; both within the fp32 contract
    w = workloads.make(cfg, n)
    ref = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)
    e = rel(fp32_op(w).apply(w.v), ref)
    assert e <= TOL32, e
    assert (e <= 1e-10) == (cfg == 2), e


@pytest.mark.parametrize("kernels", ["tf32", "ffma"])
def test_fp32_without_duplicate_merge(oracle_lib, monkeypatch, kernels):
    monkeypatch.setenv("KSVM_NFFT_F32", "all")
    monkeypatch.setenv("KSVM_NFFT_F32K", kernels)
    # config 4's binary windows at full cell density (one cell holds ~7 % of
    # the points): heavy-cell item splitting and long same-cell runs
    monkeypatch.setenv("KSVM_NFFT_DEDUP", "0")
    w = workloads.make(4, 40000)
    ref = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)
    assert rel(fp32_op(w).apply(w.v), ref) <= TOL32


@pytest.mark.parametrize("N", [8, 16, 24])
def test_fp32_wrapped_and_small_grids(oracle_lib, monkeypatch, N):
    monkeypatch.setenv("KSVM_NFFT_F32", "all")
    # N = 8, 16: the data-range grid wraps modulo M (L > M); 24: M = 48
    pts = oracle.random_points(3000, 6, 91)
    v = oracle.random_vector(3000, 92)
    wins = [[0, 1, 2], [3, 4, 5]]
    cfg = FastsumConfig(N, 4, 2, 0.25)
    g = anova_fast_operator(Dataset(pts), spec_of(wins, [1.0, 0.7]), cfg, precision="fp32")
    o = oracle_lib.anova(pts, wins, [0.5, 0.5], [1.0, 0.7], N=N, m=4, sigma=2)
    assert rel(g.apply(v), o.apply(v)) <= TOL32


def test_fp32_bit_identical_reuse_and_batch(monkeypatch):
    monkeypatch.setenv("KSVM_NFFT_F32", "all")
    # P:tests/test_fastsum.cpp:208-215 (determinism) in fp32 mode, and the
    # batched multi-RHS apply equal to single applies
    w = workloads.config2(n=20000)
    op = fp32_op(w)
    a, b = op.apply(w.v), op.apply(w.v)
    assert np.array_equal(a, b)
    V = np.stack([w.v, -0.5 * w.v, np.roll(w.v, 7)], axis=1)
    Y = op.apply_batch(V)
    for j in range(V.shape[1]):
        assert np.array_equal(Y[:, j], op.apply(np.ascontiguousarray(V[:, j])))


def test_fp32_only_touches_three_feature_windows(oracle_lib):
    # d <= 2 windows stay fp64: an operator of 1-/2-feature windows is exact
    pts = oracle.random_points(2000, 3, 95)
    v = oracle.random_vector(2000, 96)
    wins = [[0, 1], [2]]
    g = anova_fast_operator(Dataset(pts), spec_of(wins), precision="fp32")
    o = oracle_lib.anova(pts, wins)
    assert rel(g.apply(v), o.apply(v)) <= 1e-10


def test_precision_argument_checked():
    w = workloads.config1()
    with pytest.raises(ValueError):
        anova_fast_operator(Dataset(w.points), spec_of(w.windows), precision="fp16")
