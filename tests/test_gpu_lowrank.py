"""GPU: greedy pivoted Cholesky vs the oracle restatement
of P:src/low_rank.cpp:25-92 (pinned to the reference's low-rank tests in
tests/test_oracle_lowrank.py), on the same exact entries.

Bar: identical pivot sequence; factor rows within 1e-10 absolute (entries
are exp() on the device vs libm, ~1 ulp apart, propagated through the
triangular updates); trace residual within 1e-9 relative.
"""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FeatureWindowing, SaddleOperator,
                                   SaddlePreconditioner, anova_fast_operator, gmres_solve, pivoted_cholesky_greedy,
                                   stack_anova_factors)

pytestmark = pytest.mark.gpu


def make(n, seed, wins, ells=None):
    pts = oracle.random_points(n, max(f for w in wins for f in w) + 1, seed)
    P = len(wins)
    ells = ells or [1.0] * P
    spec = AnovaKernelSpec(FeatureWindowing([list(w) for w in wins], [1.0 / P] * P, ells))
    return pts, anova_fast_operator(Dataset(pts), spec), ells


@pytest.mark.parametrize("window", [0, 1, -1])
def test_matches_oracle(window):
    wins = [[0, 1, 2], [3, 4]]
    pts, op, ells = make(3000, 41, wins, [1.0, 1.7])
    f = pivoted_cholesky_greedy(op, 40, 0.0, window=window)
    Zo, tro, po = oracle.pivoted_cholesky(pts, wins, window=window, rank=40, ells=ells)
    assert f.achieved_rank == 40 and list(f.pivots) == list(po)
    assert np.abs(f.Z - Zo).max() <= 1e-10
    assert f.trace_residual == pytest.approx(tro, rel=1e-9)


def test_stop_rule_and_clamp():
    wins = [[0, 1]]
    pts, op, _ = make(500, 4, wins, [2.0])
    f = pivoted_cholesky_greedy(op, 500, 1e-5, window=0)
    Zo, tro, po = oracle.pivoted_cholesky(pts, wins, window=0, rank=500, err_tol=1e-5, ells=[2.0])
    assert f.achieved_rank == Zo.shape[0] < 500 and list(f.pivots) == list(po)
    K = oracle.dense_gaussian(pts[:, :2], 2.0)
    assert np.diag(K - f.Z.T @ f.Z).max() <= 1e-5 * (1 + 1e-10)
    g = pivoted_cholesky_greedy(op, 10 ** 6, 0.0, window=0)  # rank > n clamps to n
    assert g.achieved_rank <= 500
    with pytest.raises(ValueError):
        pivoted_cholesky_greedy(op, 0)
    with pytest.raises(ValueError):
        pivoted_cholesky_greedy(op, 5, window=3)


def test_duplicate_points_stop_at_distinct_count():
    # a binary window has 8 distinct points: the residual vanishes after 8 pivots
    rng = np.random.default_rng(3)
    X = np.hstack([rng.standard_normal((4000, 3)), (rng.random((4000, 3)) < 0.3).astype(float)])
    X = (X - X.min(0)) / (X.max(0) - X.min(0)) * 0.5 - 0.25
    wins = [[0, 1, 2], [3, 4, 5]]
    op = anova_fast_operator(Dataset(X), AnovaKernelSpec(FeatureWindowing.explicit(wins)))
    f = pivoted_cholesky_greedy(op, 30, 1e-12, window=1)
    Zo, _, po = oracle.pivoted_cholesky(X, wins, window=1, rank=30, err_tol=1e-12)
    assert f.achieved_rank == Zo.shape[0] == 8 and list(f.pivots) == list(po)


def test_factor_preconditions_gmres_end_to_end():
    # test_saddle.cpp:229-252 on the GPU: Cholesky -> stacked Z -> SMW -> GMRES
    n = 3000
    wins = [[0, 1, 2], [3, 4, 5]]
    pts, op, _ = make(n, 23, wins)
    y = np.array([1.0 if i % 2 == 0 else -1.0 for i in range(n)])
    theta = np.abs(oracle.random_vector(n, 24)) * 0.05 + 0.01
    rhs = oracle.random_vector(n + 1, 25)
    A = SaddleOperator(op, y, theta)

    def its(rank):
        if rank == 0:
            P = SaddlePreconditioner(None, y)
        else:
            fs = [pivoted_cholesky_greedy(op, rank, 0.0, window=l) for l in range(2)]
            P = SaddlePreconditioner(stack_anova_factors(fs, [0.5, 0.5]), y)
        P.refresh(theta)
        x, st = gmres_solve(A, P, rhs, 1e-8, 400)
        assert st.converged
        return st.iterations

    plain, it20, it80 = its(0), its(20), its(80)
    assert it80 < it20 < plain
