"""CPU: the reference's OWN host driver (oracle/_ref/libdriver_cpu.so:
P:src/{dataset,windowing,kernel,fastsum,low_rank,saddle,ipm,pipeline}.cpp
compiled unmodified by path against oracle/shim2) pins the oracle
restatements the GPU tests compare with (oracle/saddle_oracle.cpp,
lowrank_oracle.cpp, nystrom_oracle.cpp, dataset_oracle.cpp): on BASELINE
config 1 end to end (split, z-score, rank-50 factor, IPM with C = 1, bias,
fast prediction) both give the same Newton trajectory, GMRES iteration count
per step, dual objective, alpha and held-out decision values.

Both sides evaluate the same NFFT operator up to summation order (the
restatement is bit-identical to the reference's fastsum, tests/test_oracle.py;
the shim's dense algebra is sequential where Eigen vectorises), so the bars
are rounding-level: alpha 1e-6 (GMRES stops at a 1e-3 residual), dual
objective 1e-9, decision values 1e-6.
"""
import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import workloads
from pipeline_oracle import oracle_pipeline

pytestmark = pytest.mark.skipif(not oracle.Driver.available("cpu"),
                                reason="oracle/_ref/libdriver_cpu.so not built (needs /root/reference)")


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("precond", ["cholesky-greedy", "nystrom-gaussian"])
def test_reference_driver_pins_oracle_pipeline_config1(precond):
    w = workloads.config1()
    ref = oracle.Driver("cpu").train_steps(w.points, w.labels, w.windows, precond, 50, 1.0, 0)
    ours = oracle_pipeline(w, w.windows, 50, 1.0, precond=precond)
    assert ref["n_train"] == len(ours["tr"]) and ref["n_test"] == len(ours["te"])
    assert ref["rank"] == ours["Z"].shape[0]
    assert ref["status"] == 0 and ours["res"]["status"] == "converged"
    assert ref["ipm_iters"] == ours["res"]["iterations"]
    assert [int(x) for x in ref["log"][:, 4]] == [int(x) for x in ours["log"][:, 4]]
    assert np.allclose(ref["log"][:, 0], ours["log"][:, 0], rtol=1e-14)  # mu schedule
    assert rel(ours["alpha"], ref["alpha"]) <= 1e-6
    ya = ours["ytr"] * ours["alpha"]
    dual_o = ours["alpha"].sum() - 0.5 * ya @ ours["Ko"].apply(ya)
    assert abs(dual_o - ref["dual_objective"]) <= 1e-9 * abs(ref["dual_objective"])
    assert abs(ours["bias"] - ref["bias"]) <= 1e-6
    assert rel(ours["f"], ref["test_decision"]) <= 1e-6
    assert (np.sign(ours["f"]) == np.sign(ref["test_decision"])).mean() >= 0.999


def test_reference_train_pipeline_equals_its_steps():
    """drv_train_steps calls the functions train_pipeline calls, in its order:
    the same bits come out (the per-step log is then the reference's own)."""
    pts, y = oracle.blobs(600, 4, 2.0, 7)
    d = oracle.Driver("cpu")
    a = d.train_pipeline(pts, y, [[0, 1], [2, 3]], "cholesky-greedy", 20, 1.0, 3)
    b = d.train_steps(pts, y, [[0, 1], [2, 3]], "cholesky-greedy", 20, 1.0, 3)
    for k in ("n_train", "n_test", "ipm_iters", "status", "rank"):
        assert a[k] == b[k]
    assert a["mean_gmres"] == b["mean_gmres"] and a["dual_objective"] == b["dual_objective"]
    assert np.array_equal(a["alpha"], b["alpha"]) and np.array_equal(a["test_decision"], b["test_decision"])


def test_reference_gmres_matches_oracle_gmres():
    """gmres_solve + SaddlePreconditioner (P:src/saddle.cpp:35-178) of the
    reference against the restatement, on one Newton system of config 1's
    shape with a rank-20 greedy-Cholesky factor."""
    w = workloads.config1(n=600)
    X = w.points
    rng = np.random.default_rng(4)
    y = np.where(rng.random(600) < 0.5, 1.0, -1.0)
    theta = rng.uniform(0.5, 4.0, 600)
    rhs = rng.standard_normal(601)
    Zs = [oracle.pivoted_cholesky(X, w.windows, window=l, rank=10, err_tol=1e-5)[0] for l in range(2)]
    Z = np.vstack([np.sqrt(0.5) * z for z in Zs])
    x_ref, st = oracle.Driver("cpu").gmres(X, w.windows, y, theta, Z, rhs, 1e-8, 200)
    Ko = oracle.Lib("oracle").anova(X, w.windows, fit=1.0 / 1.2)
    x_o, st_o = oracle.gmres_solve(Ko, y, theta, Z, rhs, 1e-8, 200)
    assert st["converged"] and abs(st["iterations"] - st_o["iterations"]) <= 1
    assert rel(x_o, x_ref) <= 1e-7
