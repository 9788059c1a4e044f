"""GPU: prediction (TrainedModel::decision_values) vs the
restatement in oracle.decision_values (pinned to the reference build in
tests/test_oracle_predict.py). Bar: fast backend 1e-10 relative (the cross
transform's parity bar), exact backend 1e-12 relative, same fallback set."""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import AnovaKernelSpec, FeatureWindowing, decision_values

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("n,t", [(300, 50), (20000, 3000)])
def test_predict_matches_oracle(n, t):
    train = oracle.random_points(n, 5, 37)
    coeff = oracle.random_vector(n, 39) * 0.1
    tests = oracle.random_points(t, 5, 38)
    tests[0] = [50.0, -50.0, 3.0, 1.0, 0.0]
    tests[1] *= 4.0
    wins, w, ells = [[0, 1, 2], [3, 4]], [0.5, 0.5], [1.0, 1.3]
    spec = AnovaKernelSpec(FeatureWindowing(wins, w, ells))
    ff, nf = decision_values(train, spec, coeff, 0.25, tests, "fast")
    fo, no = oracle.decision_values(train, wins, w, ells, coeff, 0.25, tests, fast=True)
    assert nf == no >= 1
    assert rel(ff, fo) <= 1e-10
    if n <= 300:
        fe, ne = decision_values(train, spec, coeff, 0.25, tests, "exact")
        feo, _ = oracle.decision_values(train, wins, w, ells, coeff, 0.25, tests, fast=False)
        assert ne == t and rel(fe, feo) <= 1e-12
        assert np.abs(fe - ff).max() <= 1e-4 * (1.0 + np.linalg.norm(fe))


def test_predict_argument_errors():
    spec = AnovaKernelSpec(FeatureWindowing([[0, 1]], [1.0], [1.0]))
    with pytest.raises(ValueError):
        decision_values(np.zeros((10, 2)), spec, np.zeros(10), 0.0, np.zeros((3, 3)))
    with pytest.raises(ValueError):
        decision_values(np.zeros((10, 2)), spec, np.zeros(9), 0.0, np.zeros((3, 2)))
    f, ne = decision_values(np.zeros((10, 2)), spec, np.ones(10), 1.5, np.zeros((0, 2)))
    assert f.shape == (0,) and ne == 0
