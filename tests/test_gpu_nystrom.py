"""GPU: the Nystrom factor (csrc/nystrom.cu) vs the oracle restatement of
P:src/low_rank.cpp:115-168 (oracle/nystrom_oracle.cpp, pinned to
P:tests/test_low_rank.cpp:109-165 in tests/test_oracle_lowrank.py).

Columns mode uses exact kernel columns and the same LDLT on both sides:
Z agrees to rounding (1e-12). The Gaussian mode sketches the
FastWindowOperator with the reference's draws; the GPU's orthonormal basis of
range(Y) (Gram-Schmidt) and the oracle's (Householder) differ by column
signs, so the comparison is on Z^T Z, the only thing the preconditioner
uses (1e-9 relative)."""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator,
                                   fast_window_operator, nystrom)

pytestmark = pytest.mark.gpu


def gram_rel(Z, Zo, seed=0):
    x = np.random.default_rng(seed).standard_normal((Z.shape[1], 4))
    a, b = Z.T @ (Z @ x), Zo.T @ (Zo @ x)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,feats,rank,seed", [(1500, [0, 1, 2], 15, 3), (3000, [1, 3], 25, 7), (800, [2], 8, 11)])
def test_gaussian_sketch_matches_oracle(n, feats, rank, seed):
    pts = oracle.random_points(n, 4, seed) * 0.7
    fop = fast_window_operator(pts, feats, 1.0)
    f = nystrom(fop, rank, "gaussian", seed)
    Zo = oracle.nystrom_window(pts, feats, 1.0, rank, oracle.NYSTROM_GAUSSIAN, seed)
    assert f.Z.shape == Zo.shape == (rank, n)
    assert gram_rel(f.Z, Zo) <= 1e-9


@pytest.mark.parametrize("window", [0, 1])
def test_columns_sketch_matches_oracle(window):
    pts = oracle.random_points(1200, 5, 21)
    wins = [[0, 1, 2], [3, 4]]
    spec = AnovaKernelSpec(FeatureWindowing(wins, [0.5, 0.5], [1.0, 1.3]))
    op = anova_fast_operator(Dataset(pts), spec)
    f = nystrom(op, 20, "columns", 5, window=window)
    Zo = oracle.nystrom_window(pts, wins[window], [1.0, 1.3][window], 20, oracle.NYSTROM_COLUMNS, 5)
    assert np.allclose(f.Z, Zo, rtol=0, atol=1e-11 * np.abs(Zo).max())


def test_nystrom_validation_and_determinism():
    pts = oracle.random_points(50, 2, 1)
    fop = fast_window_operator(pts, [0, 1], 1.0)
    for rank in (0, 51):
        with pytest.raises(ValueError):
            nystrom(fop, rank, "gaussian", 0)
    with pytest.raises(ValueError):
        nystrom(fop, 5, "gaussian", 0, window=0)
    a, b = nystrom(fop, 6, "gaussian", 5), nystrom(fop, 6, "gaussian", 5)
    assert np.array_equal(a.Z, b.Z)


def test_device_output():
    import torch
    pts = oracle.random_points(700, 3, 2)
    fop = fast_window_operator(pts, [0, 1, 2], 1.0)
    Zd = nystrom(fop, 10, "gaussian", 9, on_device=True)
    torch.cuda.synchronize()
    assert np.array_equal(Zd.Z.cpu().numpy(), nystrom(fop, 10, "gaussian", 9).Z)
