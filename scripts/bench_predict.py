"""Measurement of GPU prediction: decision_values with the
fast backend on the BASELINE config-3 shape (train = first n/2 points, test =
the other half, as the IPM's train_fraction 0.5 split; z-scored inputs are
stood in by the workload's [-1/4, 1/4] scaling), coeff ~ N(0, 1) * 0.01.
GPU: host wall clock of the synchronous call (plans + cross transforms +
exact fallback). CPU: the oracle restatement on a bounded sample (one
window's plan + cross transform), scaled by the window count. One JSON line."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import time

import numpy as np

import oracle
from paper_2312_00538_b200 import AnovaKernelSpec, FeatureWindowing, decision_values, workloads

w = workloads.make(3)
h = w.n // 2
train, test = w.points[:h], w.points[h:]
coeff = np.random.default_rng(5).standard_normal(h) * 0.01
spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
decision_values(train, spec, coeff, 0.1, test[:1000])  # warm-up
best = 1e30
for _ in range(3):
    t0 = time.perf_counter()
    f, nex = decision_values(train, spec, coeff, 0.1, test)
    best = min(best, time.perf_counter() - t0)
win = w.windows[0]
t0 = time.perf_counter()
plan = oracle.Lib("oracle").plan(train[:, win], 1.0, fit=1 / 1.2)
sc = plan.scale_points(test[:, win])
ok = np.sqrt((sc * sc).sum(1)) <= 0.25
plan.apply_cross(test[ok][:, win], coeff)
cpu_one = time.perf_counter() - t0
P = len(w.windows)
print(json.dumps({
    "metric": "fast predictions/sec (fp64)", "value": len(test) / best, "unit": "test points/s",
    "s_per_call": best, "n_train": h, "n_test": len(test), "exact_fallback": nex,
    "config": {"workload": w.name + " predict", "windows": w.windows, "fit_fraction": 1 / 1.2,
               "timing": "host wall clock around the synchronous call (host arrays in and out)"},
    "cpu_baseline": {"value": len(test) / (cpu_one * P), "unit": "test points/s", "cores": 1, "kind": "port",
                     "sample": f"oracle plan + cross transform of window 0 ({cpu_one:.2f} s) x {P} windows"}}))
