"""Fixtures from the reference's OWN host driver (oracle/_ref/libdriver_cpu.so:
P:src/{dataset,windowing,kernel,fastsum,low_rank,saddle,ipm,pipeline}.cpp
compiled unmodified by path), run once on the CPU of the build container:

  drv_cfg3_full.npz   BASELINE config 3 at full size (n = 100000,
                             n_train ~ 5e4), Nystrom-Gaussian rank 200, C = 1
  drv_cfg5_n176k.npz  BASELINE config 5's shape at n = 176000
                             (n_train = 64238), greedy Cholesky rank 200, C = 1
  drv_cfg5_n500k.npz  the same at n = 500000 (n_train = 229246), where the
                             GPU pipeline hits the reference's stall rule

  python tests/golden/make_ref_driver_golden.py cfg3|cfg5|cfg5_500k

Each stores the split sizes, the per-Newton-step log (mu, xi_alpha_rel,
xi_lambda_rel, step_alpha, GMRES iterations, GMRES converged), status, rank,
dual objective, bias, lambda, alpha and the held-out decision values.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2312_00538_b200 import workloads  # noqa: E402

CASES = {"cfg3": (3, None, "nystrom-gaussian", "drv_cfg3_full.npz"),
         "cfg5": (5, 176000, "cholesky-greedy", "drv_cfg5_n176k.npz"),
         "cfg5_500k": (5, 500000, "cholesky-greedy", "drv_cfg5_n500k.npz")}


def main(which):
    cfg, n, precond, name = CASES[which]
    w = workloads.make(cfg, n)
    t0 = time.perf_counter()
    r = oracle.Driver("cpu").train_steps(w.points, w.labels, w.windows, precond, 200, 1.0, 0)
    secs = time.perf_counter() - t0
    np.savez_compressed(os.path.join(HERE, name), cfg=cfg, n=w.n, precond=precond, rank_req=200, seconds=secs,
                        n_train=r["n_train"], n_test=r["n_test"], ipm_iters=r["ipm_iters"], status=r["status"],
                        rank=r["rank"], dual=r["dual_objective"], bias=r["bias"], lam=r["lambda"],
                        mu_final=r["mu_final"], log=r["log"], alpha=r["alpha"], f=r["test_decision"])
    print(which, f"{secs:.1f} s", {k: v for k, v in r.items() if not isinstance(v, np.ndarray)}, r["log"][:, 4])


if __name__ == "__main__":
    main(sys.argv[1])
