"""Measurement of the batched multi-RHS apply: k = 32
columns through ksvm_nfft_op_apply_batch (device-resident), for 1, 2 and 4
apply lanes, on a BASELINE config (default 2). One JSON line; the value is
the 4-lane throughput."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import json
import os
import time

import numpy as np
import torch

from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, workloads

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--k", type=int, default=32)
args = ap.parse_args()
w = workloads.make(args.config)
op = anova_fast_operator(Dataset(w.points), AnovaKernelSpec(FeatureWindowing.explicit(w.windows)),
                         fit_fraction=w.fit_fraction)
V = torch.from_numpy(np.random.default_rng(1).standard_normal((w.n, args.k))).cuda()
res = {}
for lanes in (1, 2, 4):
    os.environ["KSVM_NFFT_LANES"] = str(lanes)
    op.apply_batch(V)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        op.apply_batch(V)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) * 1e-3)
    res[lanes] = args.k / best
print(json.dumps({"metric": "batched ANOVA-NFFT matvecs/sec (fp64)", "value": res[4], "unit": "matvecs/s",
                  "k": args.k, "by_lanes": res,
                  "config": {"workload": w.name, "n": w.n, "windows": w.windows, "fit_fraction": w.fit_fraction,
                             "timing": "CUDA events around apply_batch on device-resident V (best of 5)"}}))
