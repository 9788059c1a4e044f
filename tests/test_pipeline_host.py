"""CPU: the host side of the training pipeline (paper_2312_00538_b200.pipeline)
against the reference's own P:src/dataset.cpp (oracle/_ref) and its
restatement (oracle/dataset_oracle.cpp): the split is bit-identical (same
libstdc++ std::mt19937_64 / std::shuffle stream), the z-score equal to
rounding; window-spec parsing and config errors mirror P:src/pipeline.cpp."""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (Dataset, IpmConfig, PipelineConfig, balance_and_split, parse_window_spec,
                                   zscore_fit_transform)
from paper_2312_00538_b200 import workloads


def _labels(n, p, seed):
    rng = np.random.default_rng(seed)
    return np.where(rng.random(n) < p, 1.0, -1.0)


@pytest.mark.parametrize("n,p,frac,seed", [(2000, 0.5, 0.5, 0), (2001, 0.37, 0.5, 7), (157, 0.8, 0.3, 1001),
                                           (10, 0.5, 0.5, 3)])
def test_split_is_the_references(n, p, frac, seed, ref_lib):
    lab = _labels(n, p, seed)
    pts = np.arange(n, dtype=np.float64)[:, None] * np.ones((1, 2))
    tr, te = balance_and_split(Dataset(pts, lab), frac, seed)
    rtr, rte = oracle.balance_and_split(lab, frac, seed, "ref")
    otr, ote = oracle.balance_and_split(lab, frac, seed, "oracle")
    assert np.array_equal(tr.points[:, 0].astype(np.int64), rtr)
    assert np.array_equal(te.points[:, 0].astype(np.int64), rte)
    assert np.array_equal(otr, rtr) and np.array_equal(ote, rte)
    assert np.array_equal(tr.labels, lab[rtr]) and (tr.labels > 0).sum() == (tr.labels < 0).sum()


def test_split_errors():
    with pytest.raises(RuntimeError):  # DataError -> status 2
        balance_and_split(Dataset(np.zeros((4, 1)), np.ones(4)), 0.5, 0)
    with pytest.raises(RuntimeError):
        balance_and_split(Dataset(np.zeros((4, 1)), np.array([1.0, -1, 1, -1])), 1.0, 0)


def test_zscore_matches_reference(ref_lib):
    rng = np.random.default_rng(5)
    X = rng.normal(2.0, 3.0, size=(700, 5))
    X[:, 3] = 1.5  # constant column -> sd 1
    T = rng.normal(size=(90, 5))
    tr, te = Dataset(X.copy()), Dataset(T.copy())
    stats = zscore_fit_transform(tr, te)
    rx, rt, mu, sd = oracle.zscore(X, T, "ref")
    assert np.allclose(tr.points, rx, rtol=0, atol=1e-14) and np.allclose(te.points, rt, rtol=0, atol=1e-14)
    assert np.allclose([s.mean for s in stats], mu, rtol=1e-15) and np.allclose([s.stddev for s in stats], sd,
                                                                               rtol=1e-15)
    assert stats[3].stddev == 1.0


def test_parse_window_spec():  # P:src/pipeline.cpp:28-52
    assert parse_window_spec("0,1,2;3,4", 5) == [[0, 1, 2], [3, 4]]
    assert parse_window_spec("0,,1;;2", 3) == [[0, 1], [2]]
    for bad in ("0,x", "0,5", ";", ""):
        with pytest.raises(ValueError):
            parse_window_spec(bad, 5)


def test_config1_prepared_shapes():
    w = workloads.config1()
    tr, te = balance_and_split(Dataset(w.points, w.labels), 0.5, 0)
    assert tr.n() <= 1000 and te.n() == 1000 and tr.dim() == 6
    cfg = PipelineConfig(explicit_windows=[[0, 1, 2], [3, 4, 5]], rank=50, ipm=IpmConfig(C=1.0))
    assert cfg.ipm.C == 1.0 and cfg.precond == "cholesky-greedy"
