"""End-to-end training measurement (north_star: IPM training on the B200
path): BASELINE config 1 (n=2000, d=6, pivoted Cholesky rank 50), config 3
(n=1e5, d=22, 7x3+1 windows, Nystrom-Gaussian rank 200) and config 5
(n=1e7, d=28, 9x3+1 windows) through train_pipeline, wall clock, plus
per-phase times and the IPM trajectory. --oracle also times the CPU oracle
pipeline (config 1 only by default)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2312_00538_b200 import Dataset, IpmConfig, PipelineConfig, train_pipeline, workloads  # noqa: E402


def run(cfgno, rank, oracle_too, precond):
    w = {1: workloads.config1, 3: workloads.config3, 5: workloads.config5}[cfgno]()
    pc = PipelineConfig(explicit_windows=w.windows, rank=rank, precond=precond, ipm=IpmConfig(C=1.0))
    train_pipeline(Dataset(w.points[:400], w.labels[:400]), pc)  # warm-up (context, module load)
    t0 = time.perf_counter()
    model, test, rep, res = train_pipeline(Dataset(w.points, w.labels), pc)
    t_fit = time.perf_counter() - t0
    raw_test = test.points * np.array([s.stddev for s in model.normalization]) + np.array(
        [s.mean for s in model.normalization])
    t1 = time.perf_counter()
    pred = model.predict(raw_test)
    t_pred = time.perf_counter() - t1
    out = {"config": cfgno, "precond": precond, "n": w.points.shape[0], "n_train": rep.n_train, "n_test": rep.n_test, "rank": rep.rank,
           "train_pipeline_s": t_fit, "precond_setup_s": rep.precond_setup_seconds, "ipm_iters": rep.ipm_iters,
           "mean_gmres": rep.mean_gmres, "status": rep.status.name, "gmres_per_ipm": [
               i.gmres.iterations for i in res.iterations], "predict_s": t_pred, "phase_s": rep.phase_seconds,
           "test_accuracy": float((pred == test.labels).mean()), "bias": model.bias,
           "n_support": int(model.support_indices.size)}
    if oracle_too:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
        from test_gpu_ipm import oracle_pipeline
        t2 = time.perf_counter()
        ref = oracle_pipeline(w, w.windows, rank, 1.0, precond=precond)
        out["oracle_pipeline_s"] = time.perf_counter() - t2
        out["oracle_gmres_per_ipm"] = [int(x) for x in ref["log"][:, 4]]
        out["label_agreement_vs_oracle"] = float((np.where(ref["f"] >= 0, 1.0, -1.0) == pred).mean())
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--rank", type=int, default=None)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--precond", default=None, help="default: BASELINE's (cholesky-greedy cfg1/5, nystrom-gaussian cfg3)")
    a = ap.parse_args()
    pre = a.precond or ("nystrom-gaussian" if a.config == 3 else "cholesky-greedy")
    print(json.dumps(run(a.config, a.rank or (50 if a.config == 1 else 200), a.oracle, pre)))
