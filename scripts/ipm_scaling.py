"""Config-5-shaped IPM training (greedy Cholesky rank 200, C = 1) at growing n
on the GPU pipeline: GMRES iterations per Newton step and the IPM status at
each size. The reference's own driver reproduces the n = 176 000 run step
for step (tests/test_gpu_ref_driver.py, fixture drv_cfg5_n176k.npz); this
sweep shows how the iteration counts grow with n_train at a fixed
preconditioner rank up to BASELINE's n = 10^7, where the IPM hits the
reference's stall rule (P:src/ipm.cpp:145-149).

  python scripts/ipm_scaling.py [n ...]   -> one JSON line per n
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KSVM_NFFT_QUIET", "1")

from paper_2312_00538_b200 import Dataset, IpmConfig, PipelineConfig, train_pipeline, workloads  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [176000, 500000, 1000000, 2000000, 4000000, 10000000]
pc = None
for n in sizes:
    w = workloads.make(5, n)
    pc = PipelineConfig(explicit_windows=w.windows, rank=200, precond="cholesky-greedy", ipm=IpmConfig(C=1.0))
    if n == sizes[0]:
        train_pipeline(Dataset(w.points[:400], w.labels[:400]), pc)  # warm-up
    t0 = time.perf_counter()
    model, test, rep, res = train_pipeline(Dataset(w.points, w.labels), pc)
    secs = time.perf_counter() - t0
    print(json.dumps({"n": n, "n_train": rep.n_train, "status": rep.status.name, "newton_steps": rep.ipm_iters,
                      "gmres_per_step": [i.gmres.iterations for i in res.iterations],
                      "train_pipeline_s": secs}), flush=True)
    del w, model, test, res
