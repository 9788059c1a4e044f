"""CPU: the prediction restatement (oracle.decision_values, P:src/ipm.cpp:
213-288). Its fast part runs on the reference's own plan_fastsum /
scale_points / apply_fastsum_cross when kind="ref" (compiled by path), so the
restated orchestration is pinned to the reference build bit for bit; the
exact part equals a dense evaluation; and fast vs exact agree like
P:tests/test_ipm.cpp:345-361 requires."""
import numpy as np
import pytest

import oracle


def instance():
    train = oracle.random_points(300, 4, 37)
    coeff = oracle.random_vector(300, 39) * 0.1
    tests = oracle.random_points(50, 4, 38)
    tests[0] = [50.0, -50.0, 3.0, 1.0]  # outside the torus ball: exact fallback
    return train, coeff, tests, [[0, 1], [2, 3]], [0.5, 0.5], [1.0, 1.3]


@pytest.mark.skipif(not oracle.available("ref"), reason="reference build absent")
def test_fast_path_equals_reference_build():
    train, coeff, tests, wins, w, ells = instance()
    fo, no = oracle.decision_values(train, wins, w, ells, coeff, 0.25, tests, fast=True)
    fr, nr = oracle.decision_values(train, wins, w, ells, coeff, 0.25, tests, fast=True, kind="ref")
    assert no == nr >= 1 and np.array_equal(fo, fr)


def test_exact_path_equals_dense():
    train, coeff, tests, wins, w, ells = instance()
    fe, ne = oracle.decision_values(train, wins, w, ells, coeff, 0.25, tests, fast=False)
    K = sum(wl * np.exp(-((tests[:, None, win] - train[None, :, win]) ** 2).sum(-1) / (el * el))
            for win, wl, el in zip(wins, w, ells))
    assert ne == 50 and np.allclose(fe, K @ coeff + 0.25, rtol=1e-13, atol=1e-14)


def test_fast_agrees_with_exact():  # P:tests/test_ipm.cpp:345-361
    train, coeff, tests, wins, w, ells = instance()
    fe, _ = oracle.decision_values(train, wins, w, ells, coeff, 0.0, tests, fast=False)
    ff, nf = oracle.decision_values(train, wins, w, ells, coeff, 0.0, tests, fast=True)
    assert nf >= 1 and ff[0] == fe[0]
    assert np.abs(fe - ff).max() <= 1e-4 * (1.0 + np.linalg.norm(fe))
