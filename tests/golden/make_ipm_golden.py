"""Generate the end-to-end training fixtures (tests/golden/ipm_*.npz): the
oracle pipeline (split, z-score, preconditioner factor, IPM, bias, fast
prediction; restated in oracle/, pinned to the reference's own tests and its
dataset.cpp) on BASELINE config 3 / 5 shapes at reduced n. Too slow to rerun
inside the GPU test (minutes of CPU per case), so the GPU test compares
against these files. Run from the repo root:

    python tests/golden/make_ipm_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from paper_2312_00538_b200 import workloads  # noqa: E402
from test_gpu_ipm import oracle_pipeline  # noqa: E402

CASES = [("ipm_cfg3_n3000_nystrom.npz", 3, 3000, "nystrom-gaussian", 40),
         ("ipm_cfg5_n2500_cholesky.npz", 5, 2500, "cholesky-greedy", 40)]


def dual(alpha, y, Ko):
    ya = y * alpha
    return float(alpha.sum() - 0.5 * ya @ Ko.apply(ya))


if __name__ == "__main__":
    for name, cfg, n, pre, rank in CASES:
        w = workloads.make(cfg, n)
        r = oracle_pipeline(w, w.windows, rank, 1.0, precond=pre)
        res = r["res"]
        np.savez_compressed(os.path.join(HERE, name), cfg=cfg, n=n, precond=pre, rank=rank, tr=r["tr"], te=r["te"],
                            alpha=r["alpha"], lam=res["lambda"], xi_lambda_rel=res["xi_lambda_rel"],
                            status=res["status"], log=r["log"], bias=r["bias"], f=r["f"], zrows=r["Z"].shape[0],
                            dual=dual(r["alpha"], r["ytr"], r["Ko"]))
        print(name, res["status"], res["iterations"], [int(x) for x in r["log"][:, 4]])
