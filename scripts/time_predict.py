"""Prediction cost at a BASELINE shape: fast decision values of the held-out
split against the training split (after split + z-score), with the number of
targets that fall back to exact sums."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FeatureWindowing, balance_and_split,  # noqa: E402
                                   decision_values, workloads, zscore_fit_transform)

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = workloads.make(cfg, n)
tr, te = balance_and_split(Dataset(w.points, w.labels), 0.5, 0)
zscore_fit_transform(tr, te)
spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
coeff = np.random.default_rng(0).uniform(0, 1, tr.n()) * tr.labels
decision_values(tr.points[:1000], spec, coeff[:1000], 0.0, te.points[:1000])  # warm-up
t0 = time.perf_counter()
f, nex = decision_values(tr.points, spec, coeff, 0.0, te.points)
print(f"cfg{cfg} n_train {tr.n()} n_test {te.n()} predict {time.perf_counter() - t0:.3f} s, exact targets {nex}")
