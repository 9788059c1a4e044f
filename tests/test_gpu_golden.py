"""GPU: the B200 path against the committed golden fixtures (outputs of the
reference's own fastsum.cpp, tests/golden/make_golden.py), plus edge cases.

Tolerance: relative l2 <= 1e-10 (fp64, BASELINE.json north_star).
"""
import glob
import os

import numpy as np
import pytest

from paper_2312_00538_b200 import (AnovaKernelSpec, Dataset, DomainError, FastsumConfig,
                                   FeatureWindowing, _lib, anova_fast_operator, apply_fastsum,
                                   apply_fastsum_cross, plan_fastsum)

pytestmark = pytest.mark.gpu
TOL = 1e-10
GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "ref_*.npz")))


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def windows_of(g):
    wins, off = [], 0
    for s in g["win_sizes"]:
        wins.append([int(x) for x in g["win_features"][off:off + s]])
        off += s
    return wins


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden(path):
    g = np.load(path)
    cfg = FastsumConfig(int(g["N"]), int(g["m"]), int(g["sigma"]), float(g["rT"]))
    if str(g["kind"]) == "plan":
        p = plan_fastsum(g["points"], float(g["ell"]), cfg, float(g["fit"]))
        assert rel(apply_fastsum(p, g["v"]), g["y"]) <= TOL
        assert p.scaled_length() == float(g["scaled_length"])
        assert p.coefficient_sum() == pytest.approx(float(g["coefficient_sum"]), rel=1e-12)
        if "targets" in g:
            assert rel(apply_fastsum_cross(p, g["targets"], g["v"]), g["y_cross"]) <= TOL
    else:
        spec = AnovaKernelSpec(FeatureWindowing(windows_of(g), list(g["weights"]), list(g["ells"])))
        op = anova_fast_operator(Dataset(g["points"]), spec, cfg, float(g["fit"]))
        assert rel(op.apply(g["v"]), g["y"]) <= TOL
        assert op.entry(3, 8) == pytest.approx(float(g["entry_3_8"]), rel=1e-14)


def test_device_pointer_path_matches_host_path():
    import torch
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_cfg2_n3000.npz"))
    spec = AnovaKernelSpec(FeatureWindowing(windows_of(g), list(g["weights"]), list(g["ells"])))
    op = anova_fast_operator(Dataset(g["points"]), spec, fit_fraction=float(g["fit"]))
    host = op.apply(g["v"])
    vd = torch.from_numpy(g["v"]).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        yd = op.apply(vd)
        y2 = torch.empty_like(vd)
        op.apply_into(vd, y2)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), host)
    assert np.array_equal(y2.cpu().numpy(), host)
    assert rel(host, g["y"]) <= TOL


def test_apply_batch_equals_single_applies():
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_cfg1.npz"))
    spec = AnovaKernelSpec(FeatureWindowing(windows_of(g), list(g["weights"]), list(g["ells"])))
    op = anova_fast_operator(Dataset(g["points"]), spec, fit_fraction=float(g["fit"]))
    rng = np.random.default_rng(5)
    V = rng.standard_normal((g["points"].shape[0], 5))
    Y = op.apply_batch(V)
    for c in range(5):
        assert np.array_equal(Y[:, c], op.apply(V[:, c]))
    import torch
    Yd = op.apply_batch(torch.from_numpy(V).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(Yd.cpu().numpy(), Y)
    assert op.apply_batch(np.zeros((V.shape[0], 0))).shape == (V.shape[0], 0)
    # more columns than lanes, and an operator with duplicate-merged windows
    rng2 = np.random.default_rng(6)
    X = np.hstack([rng2.standard_normal((6000, 3)), (rng2.random((6000, 3)) < 0.2).astype(float)])
    X = (X - X.min(0)) / (X.max(0) - X.min(0)) * 0.5 - 0.25
    op2 = anova_fast_operator(Dataset(X), AnovaKernelSpec(FeatureWindowing.explicit([[0, 1, 2], [3, 4, 5]])))
    V2 = rng2.standard_normal((6000, 7))
    Y2 = op2.apply_batch(V2)
    for c in range(7):
        assert np.array_equal(Y2[:, c], op2.apply(V2[:, c]))


def test_edge_cases():
    # one point; identical points (radius 0 -> scale 1, P:src/fastsum.cpp:134); zero vector
    p = plan_fastsum(np.array([[0.1, -0.2]]), 1.0)
    assert apply_fastsum(p, np.array([2.0]))[0] == pytest.approx(2.0 * p.coefficient_sum(), rel=1e-3)
    import oracle
    z = np.zeros((5, 2))
    assert rel(apply_fastsum(plan_fastsum(z, 1.0), np.arange(5.0)),
               oracle.Lib("oracle").plan(z).apply(np.arange(5.0))) <= TOL
    pts = oracle.random_points(50, 3, 1)
    assert np.linalg.norm(apply_fastsum(plan_fastsum(pts, 1.0), np.zeros(50))) == 0.0
    # empty cross-target set; a target on the ball boundary is admissible
    p = plan_fastsum(pts, 1.0)
    assert apply_fastsum_cross(p, np.zeros((0, 3)), np.ones(50)).shape == (0,)
    s = p.scale_points(pts)
    with pytest.raises(DomainError):
        apply_fastsum_cross(p, pts * 10, np.ones(50))
    with pytest.raises(ValueError):
        apply_fastsum(p, np.ones(49))


def test_launch_counter_and_kernels_run():
    before = _lib.launch_count()
    import oracle
    pts = oracle.random_points(300, 3, 3)
    apply_fastsum(plan_fastsum(pts, 1.0), np.ones(300))
    assert _lib.launch_count() > before


def test_window_mask_partial_sums_add_up():
    # rank-local operators of the window-sharded path:
    # the partial sums over complementary window sets add up to the full apply
    from paper_2312_00538_b200 import sharding, workloads
    w = workloads.config3(n=6000)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    full = anova_fast_operator(Dataset(w.points), spec, fit_fraction=w.fit_fraction).apply(w.v)
    owner = sharding.lpt_assign(sharding.window_costs(w.windows), 3)
    total = np.zeros_like(full)
    for r in range(3):
        op = anova_fast_operator(Dataset(w.points), spec, fit_fraction=w.fit_fraction,
                                 window_mask=sharding.window_mask(owner, r))
        total += op.apply(w.v)
    assert rel(total, full) <= 1e-14
    none = anova_fast_operator(Dataset(w.points), spec, window_mask=[False] * len(w.windows))
    assert np.all(none.apply(w.v) == 0.0)
