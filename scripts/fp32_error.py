"""Relative l2 error of the fp32 mode (and of the fp64 path) against the
oracle (bit-identical to the reference's own fastsum.cpp) on BASELINE
configs 1-4 at full size and config 5 at n = 10^6."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KSVM_NFFT_QUIET", "1")
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, workloads  # noqa: E402

lib = oracle.Lib("ref") if oracle.available("ref") else oracle.Lib("oracle")
for cfg, n in ((1, None), (2, None), (3, None), (4, None), (5, 1000000)):
    w = workloads.make(cfg, n)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    ref = lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)
    out = {"config": cfg, "n": w.n}
    for prec, env in (("fp64", None), ("fp32", None), ("fp32_all", "all")):
        if env:
            os.environ["KSVM_NFFT_F32"] = env
        y = anova_fast_operator(Dataset(w.points), spec, fit_fraction=w.fit_fraction,
                                precision="fp64" if prec == "fp64" else "fp32").apply(w.v)
        os.environ.pop("KSVM_NFFT_F32", None)
        out[prec] = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
    print(json.dumps(out), flush=True)
