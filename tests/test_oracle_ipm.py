"""CPU: pin the interior point restatement (oracle.ipm_train /
compute_bias, P:src/ipm.cpp) to the reference's own tests,
P:tests/test_ipm.cpp, restated with the same instances (helpers::blobs,
DenseOperator of the exact kernel)."""
import numpy as np
import pytest

import oracle


def exact(pts, ell):
    return oracle.dense_gaussian(pts, ell)


def test_config_validation():  # :27-48
    K, y = np.eye(4), np.array([1.0, -1.0, 1.0, -1.0])
    for bad in ({"C": 0.0}, {"sigma": 1.0}, {"gamma0": 0.0}, {"tol_ip": 0.0}, {"max_ip_iters": 0}, {"mu0": -1.0}):
        with pytest.raises(oracle.OracleError):
            oracle.ipm_train(K, y, **bad)
    with pytest.raises(oracle.OracleError):  # :149-158
        oracle.ipm_train(K, np.array([1.0, -1.0, 0.5, 1.0]))


def test_converges_on_separable_blobs():  # :160-190
    pts, y = oracle.blobs(200, 2, 4.0, 11)
    K = exact(pts, 1.0)
    alpha, res, log = oracle.ipm_train(K, y)
    assert res["status"] == "converged" and res["iterations"] <= 50
    assert res["mu_final"] <= 0.1 and res["xi_alpha_rel"] <= 0.1 and res["xi_lambda_rel"] <= 0.1
    assert alpha.min() > 0.0 and alpha.max() < 0.5
    assert abs(y @ alpha) <= 1e-3 * np.abs(alpha).sum()
    b = oracle.compute_bias(K, alpha, y, 0.5, 1e-4 * 0.5)
    f = K @ (alpha * y) + b
    assert np.all(np.where(f >= 0, 1.0, -1.0) == y)


def test_barrier_schedule_and_log():  # :192-228
    pts, y = oracle.blobs(60, 2, 3.0, 13)
    alpha, res, log = oracle.ipm_train(exact(pts, 1.0), y)
    for k in range(res["iterations"]):
        assert log[k, 0] == pytest.approx(0.6 ** (k + 1), rel=1e-12)
        assert log[k, 3] > 0.0
    assert res["mu_final"] == pytest.approx(0.6 ** res["iterations"], rel=1e-12)
    assert res["xi_alpha_rel"] == log[-1, 1] and res["xi_lambda_rel"] == log[-1, 2]
    assert res["mean_gmres_iters"] == pytest.approx(log[:, 4].mean(), rel=1e-15)


def test_deterministic():  # :230-239
    pts, y = oracle.blobs(80, 2, 3.0, 19)
    K = exact(pts, 1.0)
    a1, r1, _ = oracle.ipm_train(K, y)
    a2, r2, _ = oracle.ipm_train(K, y)
    assert np.array_equal(a1, a2) and r1["lambda"] == r2["lambda"] and r1["iterations"] == r2["iterations"]


def test_preconditioned_matches_unpreconditioned():  # :241-258
    pts, y = oracle.blobs(150, 2, 3.0, 23)
    K = exact(pts, 1.0)
    Z, _, _ = oracle.pivoted_cholesky_dense(K, 60, 1e-12)
    plain, rp, _ = oracle.ipm_train(K, y)
    pre, rq, _ = oracle.ipm_train(K, y, Z)
    assert rq["status"] == "converged"
    assert np.linalg.norm(plain - pre) <= 1e-2 * np.linalg.norm(plain)
    assert rq["mean_gmres_iters"] <= rp["mean_gmres_iters"] + 1e-12


def test_bias_rules():  # :260-293
    K = np.eye(4)
    y = np.array([1.0, 1.0, -1.0, -1.0])
    assert oracle.compute_bias(K, np.array([0.4, 1.0, 0.2, 0.0]), y, 1.0, 1e-4) == pytest.approx(
        0.5 * ((1.0 - 0.4) + (-1.0 * (1.0 - 0.2))), rel=1e-14)
    assert oracle.compute_bias(K, np.array([1.0, 1.0, 1.0, 0.0]), y, 1.0, 1e-4) == pytest.approx(0.0, abs=1e-15)
    assert oracle.compute_bias(np.zeros((4, 4)), np.array([1.0, 1.0, 1.0, 0.0]), y, 1.0, 1e-4) == pytest.approx(1.0)
    assert oracle.compute_bias(K, np.zeros(4), y, 1.0, 1e-4) == 0.0
