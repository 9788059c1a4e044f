"""Generate the committed golden fixtures under tests/golden/.

Runs the REFERENCE's own hot-path code (oracle/_ref/libref.so: the unmodified
/root/reference/proj/src/fastsum.cpp + kernel.cpp + windowing.cpp compiled by
path against oracle/shim) on small seeded inputs and stores inputs and outputs
as .npz. Inputs follow the reference's test helpers (libstdc++ mt19937_64 +
normal_distribution, P:tests/helpers.hpp:15-31) and the BASELINE configs at
reduced n. Run in a container that has /root/reference (the fixtures travel;
the reference does not):

    make -C oracle && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2312_00538_b200 import workloads  # noqa: E402


def plan_case(R, name, pts, v, ell=1.0, N=32, m=4, sigma=2, rT=0.25, fit=1.0, targets=None):
    p = R.plan(pts, ell, N, m, sigma, rT, fit)
    out = dict(kind="plan", points=pts, v=v, ell=ell, N=N, m=m, sigma=sigma, rT=rT, fit=fit,
               y=p.apply(v), scaled_length=p.scaled_length(), coefficient_sum=p.coefficient_sum())
    if targets is not None:
        out["targets"] = targets
        out["y_cross"] = p.apply_cross(targets, v)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)


def anova_case(R, name, pts, v, windows, weights=None, ells=None, N=32, m=4, sigma=2, rT=0.25, fit=1.0):
    P = len(windows)
    weights = weights if weights is not None else [1.0 / P] * P
    ells = ells if ells is not None else [1.0] * P
    op = R.anova(pts, windows, weights, ells, N, m, sigma, rT, fit)
    flat = np.array([f for w in windows for f in w], dtype=np.int32)
    sizes = np.array([len(w) for w in windows], dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), kind="anova", points=pts, v=v,
                        win_features=flat, win_sizes=sizes, weights=np.array(weights),
                        ells=np.array(ells), N=N, m=m, sigma=sigma, rT=rT, fit=fit, y=op.apply(v),
                        entry_3_8=op.entry(3, 8))


def main():
    R = oracle.Lib("ref")
    # P:tests/test_fastsum.cpp inputs
    for d in (1, 2, 3):
        plan_case(R, f"ref_plan_d{d}_n500", oracle.random_points(500, d, 31), oracle.random_vector(500, 32))
    plan_case(R, "ref_plan_cross_d2", oracle.random_points(300, 2, 51), oracle.random_vector(300, 52),
              targets=oracle.random_points(100, 2, 53, 0.5))
    plan_case(R, "ref_plan_d2_N16_m4", oracle.random_points(400, 2, 71), oracle.random_vector(400, 72), N=16)
    plan_case(R, "ref_plan_d3_N8_wrap", oracle.random_points(300, 3, 73), oracle.random_vector(300, 74), N=8)
    plan_case(R, "ref_plan_d3_m6", oracle.random_points(300, 3, 75), oracle.random_vector(300, 76), m=6)
    plan_case(R, "ref_plan_d2_fit083", oracle.random_points(300, 2, 77), oracle.random_vector(300, 78),
              fit=1.0 / 1.2)
    anova_case(R, "ref_anova_n1000_d6", oracle.random_points(1000, 6, 61), oracle.random_vector(1000, 62),
               [[0, 1, 2], [3, 4, 5]], [0.5, 0.5], [1.0, 1.3])
    # BASELINE config shapes at small n
    w = workloads.config1()
    anova_case(R, "ref_cfg1", w.points, w.v, w.windows, fit=w.fit_fraction)
    for cfg, n in ((2, 3000), (3, 2000), (4, 2000), (5, 2000)):
        w = workloads.make(cfg, n)
        anova_case(R, f"ref_cfg{cfg}_n{n}", w.points, w.v, w.windows, fit=w.fit_fraction)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
