"""CPU: pin the saddle-system oracle (oracle/saddle_oracle.cpp) to the
reference's own known-answer and property tests, P:tests/test_saddle.cpp,
restated case by case with the same instances (P:tests/helpers.hpp inputs).
"""
import numpy as np
import pytest

import oracle


def alternating(n):  # helpers::alternating_labels
    return np.array([1.0 if i % 2 == 0 else -1.0 for i in range(n)])


class Inst:  # test_saddle.cpp:16-35
    def __init__(self, n, seed):
        self.K = oracle.dense_gaussian(oracle.random_points(n, 3, seed), 1.0)
        self.y = alternating(n)
        self.theta = np.abs(oracle.random_vector(n, seed + 1)) + 0.5

    def dense_saddle(self):
        n = self.y.size
        A = np.zeros((n + 1, n + 1))
        A[:n, :n] = np.diag(self.y) @ self.K @ np.diag(self.y) + np.diag(self.theta)
        A[:n, n] = -self.y
        A[n, :n] = -self.y
        return A


@pytest.mark.parametrize("n", [5, 60, 500])
def test_saddle_operator_equals_dense_block_assembly(n):  # :38-47
    inst = Inst(n, 7 + n)
    vw = oracle.random_vector(n + 1, 3)
    dense = inst.dense_saddle() @ vw
    assert np.linalg.norm(oracle.saddle_apply(inst.K, inst.y, inst.theta, vw) - dense) <= 1e-10 * np.linalg.norm(dense)


def test_null_factor_is_identity():  # :58-65
    inst = Inst(20, 2)
    g = oracle.random_vector(21, 4)
    out, _ = oracle.precond_apply(None, inst.y, inst.theta, g)
    assert np.array_equal(out, g)


def test_zero_low_rank_block_is_theta_diagonal_solve():  # :67-79
    inst = Inst(15, 3)
    g = oracle.random_vector(16, 5)
    x, _ = oracle.precond_apply(np.zeros((4, 15)), inst.y, inst.theta, g)
    x1 = g[:15] / inst.theta
    assert np.linalg.norm(x[:15] - x1) <= 1e-13 * np.linalg.norm(x1)
    assert x[15] == pytest.approx(-inst.y @ x1 - g[15], rel=1e-12)


def test_smw_matches_dense_inverse():  # :100-120
    n = 50
    inst = Inst(n, 8)
    Z = oracle.random_points(5, n, 9)
    Ahat = np.diag(inst.y) @ (Z.T @ Z) @ np.diag(inst.y) + np.diag(inst.theta)
    g = oracle.random_vector(n + 1, 10)
    x, fb = oracle.precond_apply(Z, inst.y, inst.theta, g)
    x1 = np.linalg.solve(Ahat, g[:n])
    assert not fb
    assert np.linalg.norm(x[:n] - x1) <= 1e-10 * np.linalg.norm(x1)
    assert x[n] == pytest.approx(-inst.y @ x1 - g[n], rel=1e-9)
    assert np.linalg.norm(oracle.precond_apply(Z, inst.y, inst.theta, np.zeros(n + 1))[0]) == 0.0


def test_theta_scaling_tracks_dense_inverse():  # :122-140
    n, c = 30, 4.0
    inst = Inst(n, 11)
    Z = oracle.random_points(3, n, 12)
    Ahat = np.diag(inst.y) @ (Z.T @ Z) @ np.diag(inst.y) + np.diag(c * inst.theta)
    g = oracle.random_vector(n + 1, 13)
    x1 = np.linalg.solve(Ahat, g[:n])
    assert np.linalg.norm(oracle.precond_apply(Z, inst.y, c * inst.theta, g)[0][:n] - x1) <= 1e-10 * np.linalg.norm(x1)


def test_exact_factor_converges_in_few_iterations():  # :151-183
    n = 60
    inst = Inst(n, 15)
    Z = np.linalg.cholesky(inst.K + 1e-12 * np.eye(n)).T
    rhs = oracle.random_vector(n + 1, 16)
    x, st = oracle.gmres_solve(inst.K, inst.y, inst.theta, Z, rhs, 1e-10, 100)
    assert st["converged"] and st["iterations"] <= 3
    assert np.linalg.norm(rhs - inst.dense_saddle() @ x) <= 1e-10 * np.linalg.norm(rhs)


def test_gmres_zero_rhs():  # :185-195
    inst = Inst(10, 17)
    x, st = oracle.gmres_solve(inst.K, inst.y, inst.theta, None, np.zeros(11), 1e-8, 50)
    assert np.linalg.norm(x) == 0.0 and st["iterations"] == 0 and st["converged"]


def test_gmres_residual_contract():  # :197-214
    n = 80
    inst = Inst(n, 18)
    Z = oracle.random_points(10, n, 19)
    rhs = oracle.random_vector(n + 1, 20)
    x, st = oracle.gmres_solve(inst.K, inst.y, inst.theta, Z, rhs, 1e-6, 100)
    res = np.linalg.norm(rhs - inst.dense_saddle() @ x) / np.linalg.norm(rhs)
    if st["converged"]:
        assert res <= 1e-6 * (1 + 1e-12)
    assert st["relative_residual"] == pytest.approx(res, rel=1e-10)


def test_gmres_residual_estimates_nonincreasing():  # :216-227
    n = 100
    inst = Inst(n, 21)
    rhs = oracle.random_vector(n + 1, 22)
    _, st = oracle.gmres_solve(inst.K, inst.y, inst.theta, None, rhs, 1e-12, 100)
    h = st["residual_history"]
    assert len(h) > 5 and all(h[i] <= h[i - 1] + 1e-12 for i in range(1, len(h)))


def test_preconditioning_reduces_iterations_with_rank():  # :229-252 (Cholesky factors of rank r)
    n = 400
    inst = Inst(n, 23)
    rhs = oracle.random_vector(n + 1, 24)

    def its(Z):
        return oracle.gmres_solve(inst.K, inst.y, inst.theta, Z, rhs, 1e-8, 400)[1]["iterations"]

    plain = its(None)
    # rank-r pivoted factors stand-in: leading columns of a pivoted LDL via
    # numpy (greedy pivoted Cholesky is SURVEY.md 8(f)3, not restated here)
    def pivoted(r):
        d = np.diag(inst.K).copy()
        Z = np.zeros((r, n))
        for k in range(r):
            p = int(np.argmax(d))
            row = inst.K[p] - Z[:k].T @ Z[:k, p]
            Z[k] = row / np.sqrt(d[p])
            d -= Z[k] ** 2
            d[p] = 0.0
            d = np.maximum(d, 0.0)
        return Z

    it50, it150 = its(pivoted(50)), its(pivoted(150))
    assert it150 < it50 < plain


def test_gmres_rejects_bad_arguments():
    inst = Inst(10, 1)
    with pytest.raises(oracle.OracleError):
        oracle.gmres_solve(inst.K, inst.y, inst.theta, None, np.ones(11), 0.0, 10)
    with pytest.raises(oracle.OracleError):  # Theta must be positive (P:src/saddle.cpp:42-43)
        oracle.gmres_solve(inst.K, inst.y, np.zeros(10), np.zeros((1, 10)), np.ones(11), 1e-6, 10)
