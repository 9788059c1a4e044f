"""Measurement of the GPU-resident saddle solve.

One Newton-system solve of the IPM (P:src/ipm.cpp:128 -> gmres_solve,
P:src/saddle.cpp:92-178) on a BASELINE shape: K the ANOVA NFFT operator
(fit 1/1.2 as in training), labels +-1, Theta in [0.5, 1.5), a rank-k stacked
factor Z (k = 50, seeded Gaussian, scaled so the SMW correction is active),
rhs ~ N(0, 1). Device time of the whole solve (CUDA events on the stream,
inputs resident), and the oracle restatement (CPU, 1 thread) timed on a
bounded sample (first 3 GMRES iterations), scaled to the GPU's iteration
count. Prints one JSON line.
"""
import argparse
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import time

import numpy as np
import torch

import oracle
from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, FeatureWindowing, SaddleOperator,
                                   SaddlePreconditioner, anova_fast_operator, gmres_solve, workloads)

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--rank", type=int, default=50)
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--max-iter", type=int, default=100)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--no-oracle", action="store_true")
args = ap.parse_args()

w = workloads.make(args.config, args.n)
n = w.n
rng = np.random.default_rng(7)
spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
K = anova_fast_operator(Dataset(w.points), spec, fit_fraction=1 / 1.2)
y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
theta = 0.5 + rng.random(n)
Z = rng.standard_normal((args.rank, n)) / np.sqrt(n)
rhs = rng.standard_normal(n + 1)
A = SaddleOperator(K, y, theta)
P = SaddlePreconditioner(Z, y)
t0 = time.perf_counter()
P.refresh(theta)
first_refresh_s = time.perf_counter() - t0
rts = []
for _ in range(5):  # warm refreshes (kernels loaded)
    t0 = time.perf_counter()
    P.refresh(theta)
    rts.append(time.perf_counter() - t0)
refresh_s = float(np.median(rts))
rd = torch.from_numpy(rhs).cuda()
x, st = gmres_solve(A, P, rd, args.tol, args.max_iter)  # warm-up (workspace, graphs)
torch.cuda.synchronize()
times = []
for _ in range(args.reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    x, st = gmres_solve(A, P, rd, args.tol, args.max_iter)
    e.record()
    torch.cuda.synchronize()
    times.append(s.elapsed_time(e))
gpu_ms = sorted(times)[len(times) // 2]

v1 = torch.from_numpy(w.v).cuda()
y1 = torch.empty_like(v1)
for _ in range(3):
    K.apply_into(v1, y1)
torch.cuda.synchronize()
s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s_.record()
for _ in range(10):
    K.apply_into(v1, y1)
e_.record()
torch.cuda.synchronize()
matvec_ms = s_.elapsed_time(e_) / 10
if args.no_oracle:
    print(json.dumps({"config": args.config, "n": n, "rank": args.rank, "gmres_iterations": st.iterations,
                      "solve_ms": gpu_ms, "ms_per_iteration": gpu_ms / max(st.iterations, 1),
                      "matvec_ms_back_to_back": matvec_ms, "refresh_s": refresh_s, "first_refresh_s": first_refresh_s}))
    raise SystemExit(0)
Ko = oracle.Lib("oracle").anova(w.points, w.windows, fit=1 / 1.2)
t0 = time.perf_counter()
_, so = oracle.gmres_solve(Ko, y, theta, Z, rhs, args.tol, 3)
cpu_3 = time.perf_counter() - t0
# 3 iterations cost 3 + 2 preconditioned matvecs (final x and residual); scale by matvec count
cpu_s = cpu_3 * (st.iterations + 2) / (3 + 2)
line = {"metric": "GMRES saddle solves/sec (fp64)", "value": 1e3 / gpu_ms, "unit": "solves/s",
        "ms_per_solve": gpu_ms, "iterations": st.iterations, "ms_per_iteration": gpu_ms / max(st.iterations, 1),
        "converged": st.converged, "relative_residual": st.relative_residual,
        "precond_refresh_s": refresh_s,
        "config": {"workload": w.name, "n": n, "windows": w.windows, "fit_fraction": 1 / 1.2, "rank": args.rank,
                   "tol": args.tol, "max_iter": args.max_iter, "data": "synthetic (seeded)"},
        "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "solves/s", "cores": 1, "kind": "port",
                         "sample": f"oracle restatement of P:src/saddle.cpp, first 3 GMRES iterations "
                                   f"({cpu_3:.2f} s) scaled to {st.iterations} iterations"}}
print(json.dumps(line))
