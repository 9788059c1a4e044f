"""CPU: pin the greedy pivoted Cholesky oracle (oracle/lowrank_oracle.cpp) to
the reference's own tests, P:tests/test_low_rank.cpp:20-78, restated with
the same instances (P:tests/helpers.hpp inputs)."""
import numpy as np
import pytest

import oracle


def test_identity_ties_to_smallest_index():  # :20-28
    Z, tr, piv = oracle.pivoted_cholesky_dense(np.eye(3), 2, 0.0)
    assert Z.shape == (2, 3) and list(piv) == [0, 1]
    assert np.allclose(Z, np.eye(3)[:2]) and tr == pytest.approx(1.0, rel=1e-14)


def test_rank_one_exact_after_one_pivot():  # :30-36
    z = oracle.random_vector(30, 1)
    M = np.outer(z, z)
    Z, _, _ = oracle.pivoted_cholesky_dense(M, 5, 1e-12)
    assert Z.shape[0] == 1 and np.linalg.norm(Z.T @ Z - M) <= 1e-10


def test_error_decreases_with_rank_and_trace_identity():  # :38-53
    K = oracle.dense_gaussian(oracle.random_points(300, 3, 2), 1.0)
    prev = 1e300
    for rank in (10, 20, 50):
        Z, tr, _ = oracle.pivoted_cholesky_dense(K, rank, 0.0)
        err = np.linalg.norm(Z.T @ Z - K)
        assert err < prev
        assert tr == pytest.approx(np.trace(K) - (Z ** 2).sum(), rel=1e-8)
        prev = err


def test_full_rank_reproduces():  # :55-61
    K = oracle.dense_gaussian(oracle.random_points(100, 3, 3), 1.5)
    Z, _, _ = oracle.pivoted_cholesky_dense(K, 100, 0.0)
    assert np.linalg.norm(Z.T @ Z - K) <= 1e-10 * np.linalg.norm(K)


def test_early_exit_at_err_tol():  # :63-71
    K = oracle.dense_gaussian(oracle.random_points(200, 2, 4), 2.0)
    Z, _, _ = oracle.pivoted_cholesky_dense(K, 200, 1e-5)
    assert Z.shape[0] < 200
    assert np.diag(K - Z.T @ Z).max() <= 1e-5 * (1 + 1e-10)


def test_rejects_indefinite():  # :73-78
    with pytest.raises(oracle.OracleError):
        oracle.pivoted_cholesky_dense(np.array([[1.0, 2.0], [2.0, 1.0]]), 2, 0.0)
    with pytest.raises(oracle.OracleError):
        oracle.pivoted_cholesky_dense(np.eye(2), 0, 0.0)


def test_window_entries_equal_dense_gaussian():
    # the point-based entry modes equal the dense kernels they stand for
    pts = oracle.random_points(150, 5, 8)
    Zw, trw, pw = oracle.pivoted_cholesky(pts, [[0, 1, 2], [3, 4]], window=1, rank=20)
    Zd, trd, pd = oracle.pivoted_cholesky_dense(oracle.dense_gaussian(pts[:, 3:5], 1.0), 20)
    assert list(pw) == list(pd) and np.allclose(Zw, Zd, rtol=0, atol=1e-14)
    Ka = 0.5 * oracle.dense_gaussian(pts[:, 0:3], 1.0) + 0.5 * oracle.dense_gaussian(pts[:, 3:5], 1.0)
    Za, _, pa = oracle.pivoted_cholesky(pts, [[0, 1, 2], [3, 4]], window=-1, rank=20)
    Zb, _, pb = oracle.pivoted_cholesky_dense(Ka, 20)
    assert list(pa) == list(pb) and np.allclose(Za, Zb, rtol=0, atol=1e-13)
