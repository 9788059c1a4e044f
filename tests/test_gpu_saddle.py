"""GPU: the GPU-resident saddle solver vs the oracle
restatement of P:src/saddle.cpp (oracle/saddle_oracle.cpp, pinned to the
reference's saddle tests in tests/test_oracle_saddle.py), with K the same
NFFT ANOVA operator on both sides (GPU: AnovaFastOperator; oracle: the
restated fastsum path).

Tolerances: saddle/preconditioner applies 1e-12 relative (rounding of the
operator and of fixed-order reductions); GMRES solutions 1e-8 relative
(classical vs modified Gram-Schmidt, both with one re-orthogonalisation
pass, differ by rounding that GMRES propagates through ~30 iterations).
"""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FeatureWindowing, SaddleOperator,
                                   SaddlePreconditioner, anova_fast_operator, gmres_solve)

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


class Inst:
    """test_saddle.cpp:16-35 instance with the NFFT operator for K."""

    def __init__(self, n, seed, wins=((0, 1, 2),), d=3):
        self.pts = oracle.random_points(n, d, seed)
        wins = [list(w) for w in wins]
        spec = AnovaKernelSpec(FeatureWindowing(wins, [1.0 / len(wins)] * len(wins), [1.0] * len(wins)))
        self.K = anova_fast_operator(Dataset(self.pts), spec)
        self.Ko = oracle.Lib("oracle").anova(self.pts, wins)
        self.y = np.array([1.0 if i % 2 == 0 else -1.0 for i in range(n)])
        self.theta = np.abs(oracle.random_vector(n, seed + 1)) + 0.5
        self.n = n


@pytest.mark.parametrize("n", [5, 60, 3000])
def test_saddle_apply_matches_oracle(n):
    inst = Inst(n, 7 + n)
    A = SaddleOperator(inst.K, inst.y, inst.theta)
    vw = oracle.random_vector(n + 1, 3)
    assert rel(A.apply(vw), oracle.saddle_apply(inst.Ko, inst.y, inst.theta, vw)) <= 1e-12
    assert A.size() == n + 1


# 200: SMEM-staged Gram + cluster inverse; 230: per-tile Gram + cluster
# inverse; 340: per-tile Gram + one-CTA inverse (saddle.cu)
@pytest.mark.parametrize("rank", [0, 1, 5, 40, 200, 230, 340])
def test_preconditioner_matches_oracle(rank):
    n = 2000
    inst = Inst(n, 31)
    Z = None if rank == 0 else oracle.random_points(rank, n, 9) * 0.3
    P = SaddlePreconditioner(Z, inst.y)
    assert P.identity() == (Z is None)
    for c in (1.0, 4.0):
        P.refresh(c * inst.theta)
        g = oracle.random_vector(n + 1, 10)
        want, fb = oracle.precond_apply(Z, inst.y, c * inst.theta, g)
        got = P.apply(g)
        assert P.diagonal_fallback() == fb
        if Z is None:
            assert np.array_equal(got, g)
        else:
            assert rel(got, want) <= 1e-12
    # zero block: the Theta diagonal solve (test_saddle.cpp:67-79)
    Pz = SaddlePreconditioner(np.zeros((4, n)), inst.y)
    Pz.refresh(inst.theta)
    g = oracle.random_vector(n + 1, 5)
    x = Pz.apply(g)
    x1 = g[:n] / inst.theta
    assert rel(x[:n], x1) <= 1e-13
    assert x[n] == pytest.approx(-inst.y @ x1 - g[n], rel=1e-12)


@pytest.mark.parametrize("rank", [None, 10])
def test_gmres_matches_oracle(rank):
    n = 4000
    inst = Inst(n, 18)
    Z = None if rank is None else oracle.random_points(rank, n, 19) * 0.3
    A = SaddleOperator(inst.K, inst.y, inst.theta)
    P = SaddlePreconditioner(Z, inst.y)
    P.refresh(inst.theta)
    rhs = oracle.random_vector(n + 1, 20)
    x, st = gmres_solve(A, P, rhs, 1e-8, 200)
    xo, so = oracle.gmres_solve(inst.Ko, inst.y, inst.theta, Z, rhs, 1e-8, 200)
    assert st.converged and so["converged"]
    assert abs(st.iterations - so["iterations"]) <= 1
    assert rel(x, xo) <= 1e-8
    # the true residual of the returned x (P:src/saddle.cpp:174-176)
    res = rel(oracle.saddle_apply(inst.Ko, inst.y, inst.theta, x), rhs)
    assert st.relative_residual <= 1e-8 and res <= 1e-8
    assert np.all(np.diff(st.residual_history) <= 1e-12)
    n2 = min(len(st.residual_history), len(so["residual_history"])) - 1
    assert np.allclose(st.residual_history[:n2], so["residual_history"][:n2], rtol=1e-6)


def test_exact_factor_converges_in_three_iterations():
    # test_saddle.cpp:151-183 with the exact factor of the NFFT operator K~
    n = 60
    inst = Inst(n, 15)
    Kd = np.stack([inst.Ko.apply(e) for e in np.eye(n)], axis=1)
    Kd = 0.5 * (Kd + Kd.T)
    Z = np.linalg.cholesky(Kd + 1e-12 * np.eye(n)).T
    A = SaddleOperator(inst.K, inst.y, inst.theta)
    P = SaddlePreconditioner(Z, inst.y)
    P.refresh(inst.theta)
    rhs = oracle.random_vector(n + 1, 16)
    x, st = gmres_solve(A, P, rhs, 1e-10, 100)
    assert st.converged and st.iterations <= 3
    assert rel(A.apply(x), rhs) <= 1e-10


def test_gmres_zero_rhs_and_reproducibility():
    inst = Inst(500, 17)
    A = SaddleOperator(inst.K, inst.y, inst.theta)
    P = SaddlePreconditioner(None, inst.y)
    P.refresh(inst.theta)
    x, st = gmres_solve(A, P, np.zeros(501), 1e-8, 50)
    assert np.linalg.norm(x) == 0.0 and st.iterations == 0 and st.converged
    rhs = oracle.random_vector(501, 22)
    a, sa = gmres_solve(A, P, rhs, 1e-10, 100)
    b, sb = gmres_solve(A, P, rhs, 1e-10, 100)
    assert np.array_equal(a, b) and sa.iterations == sb.iterations
    # max_iter hit: best iterate, converged false, true residual reported
    c, sc = gmres_solve(A, P, rhs, 1e-14, 3)
    assert sc.iterations == 3 and not sc.converged
    assert sc.relative_residual == pytest.approx(rel(A.apply(c), rhs), rel=1e-9)


def test_device_pointers_match_host():
    import torch
    inst = Inst(3000, 23)
    A = SaddleOperator(inst.K, inst.y, inst.theta)
    P = SaddlePreconditioner(oracle.random_points(8, 3000, 5) * 0.3, inst.y)
    P.refresh(inst.theta)
    rhs = oracle.random_vector(3001, 24)
    xh, sh = gmres_solve(A, P, rhs, 1e-9, 100)
    xd, sd = gmres_solve(A, P, torch.from_numpy(rhs).cuda(), 1e-9, 100)
    torch.cuda.synchronize()
    assert np.array_equal(xd.cpu().numpy(), xh) and sd.iterations == sh.iterations
    g = torch.from_numpy(rhs).cuda()
    assert np.array_equal(A.apply(g).cpu().numpy(), A.apply(rhs))
    assert np.array_equal(P.apply(g).cpu().numpy(), P.apply(rhs))


def test_errors_follow_the_reference():
    inst = Inst(50, 1)
    with pytest.raises(ValueError):
        SaddleOperator(inst.K, inst.y, np.zeros(50))  # P:src/saddle.cpp:12-13
    A = SaddleOperator(inst.K, inst.y, inst.theta)
    with pytest.raises(ValueError):
        A.set_theta(-np.ones(50))
    P = SaddlePreconditioner(np.zeros((1, 50)), inst.y)
    with pytest.raises(RuntimeError):
        P.apply(np.zeros(51))  # apply before refresh (P:src/saddle.cpp:70-71)
    with pytest.raises(ValueError):
        P.refresh(np.zeros(50))
    P.refresh(inst.theta)
    with pytest.raises(ValueError):
        gmres_solve(A, P, np.ones(51), 0.0, 10)
    with pytest.raises(ValueError):
        A.apply(np.ones(50))
