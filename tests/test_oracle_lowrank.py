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


# --- Nystrom (oracle/nystrom_oracle.cpp) pinned to P:tests/test_low_rank.cpp:109-165
def test_nystrom_gaussian_exact_on_rank_k():  # :109-115
    B = oracle.random_points(80, 6, 8)
    M = B @ B.T
    Z = oracle.nystrom_dense(M, 6, oracle.NYSTROM_GAUSSIAN, 3)
    assert np.linalg.norm(Z.T @ Z - M) <= 1e-8 * np.linalg.norm(M)


def test_nystrom_columns_identity_projector():  # :117-127
    Z = oracle.nystrom_dense(np.eye(12), 4, oracle.NYSTROM_COLUMNS, 11)
    P = Z.T @ Z
    assert np.linalg.norm(P @ P - P) <= 1e-10
    assert np.trace(P) == pytest.approx(4.0, rel=1e-10)
    assert all(abs(x) <= 1e-10 or abs(x - 1.0) <= 1e-10 for x in np.diag(P))


def test_nystrom_columns_reconstructs_sampled_columns():  # :129-140
    K = oracle.dense_gaussian(oracle.random_points(150, 3, 12), 1.2)
    Z = oracle.nystrom_dense(K, 20, oracle.NYSTROM_COLUMNS, 21)
    A = Z.T @ Z
    assert sum(np.linalg.norm(A[:, j] - K[:, j]) <= 1e-8 for j in range(150)) >= 20


def test_nystrom_gaussian_within_10x_of_best():  # :142-154
    K = oracle.dense_gaussian(oracle.random_points(300, 3, 13), 1.0)
    Z = oracle.nystrom_dense(K, 50, oracle.NYSTROM_GAUSSIAN, 31)
    err = np.linalg.norm(Z.T @ Z - K)
    ev = np.linalg.eigvalsh(K)
    assert err <= 10.0 * np.sqrt((ev[: 300 - 50] ** 2).sum())


def test_nystrom_validation_and_determinism():  # :156-165
    for rank, mode in ((6, oracle.NYSTROM_COLUMNS), (0, oracle.NYSTROM_GAUSSIAN)):
        with pytest.raises(oracle.OracleError):
            oracle.nystrom_dense(np.eye(5), rank, mode, 0)
    a = oracle.nystrom_dense(np.eye(5), 3, oracle.NYSTROM_GAUSSIAN, 5)
    b = oracle.nystrom_dense(np.eye(5), 3, oracle.NYSTROM_GAUSSIAN, 5)
    assert np.array_equal(a, b)


def test_nystrom_window_fast_and_exact_agree():
    """FastWindowOperator (plan fit 1.0) vs the exact WindowOperator sketch on
    the same seed: same Gaussian draw, K approximated to the NFFT error."""
    pts = oracle.random_points(400, 4, 17) * 0.5
    Zf = oracle.nystrom_window(pts, [0, 2], 1.0, 15, oracle.NYSTROM_GAUSSIAN, 4)
    K = oracle.dense_gaussian(pts[:, [0, 2]], 1.0)
    Ze = oracle.nystrom_dense(K, 15, oracle.NYSTROM_GAUSSIAN, 4)
    assert np.linalg.norm(Zf.T @ Zf - Ze.T @ Ze) <= 1e-3 * np.linalg.norm(K)
    Zc = oracle.nystrom_window(pts, [0, 2], 1.0, 15, oracle.NYSTROM_COLUMNS, 4)
    assert np.allclose(Zc, oracle.nystrom_dense(K, 15, oracle.NYSTROM_COLUMNS, 4), rtol=0, atol=1e-12)
