"""GPU: the multi-rank matvec paths, two processes on one device.

This pool grants one GPU, so the two ranks share cuda:0 and sum over gloo
(host-staged collectives, sharding.make_collectives): no rank's kernels wait
on another's, only the host-side collective joins them. What runs is the
real multi-GPU code: each rank's operator is the library's window-masked
operator (window sharding, north_star / SURVEY.md 8(e)) driven through the
pipelined apply_windows + combine_range + chunked all-reduce, or the
point-sharded operator (SURVEY.md 8(e) hybrid) with its grid pool summed by
ONE all-reduce and y assembled by ONE all-gather. Both must equal the
single-process operator to 1e-12 and the oracle to 1e-10.
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2312_00538_b200 import workloads

pytestmark = pytest.mark.gpu

CASES = {"cfg3": (3, 30000), "cfg5": (5, 60000), "cfg2": (2, 20000)}


def _worker(rank, world, port, out_dir, mode, case):
    import torch
    import torch.distributed as dist
    from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg, n = CASES[case]
    w = workloads.make(cfg, n)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    allreduce, allreduce_async, allgather = sharding.make_collectives("gloo")
    v = torch.from_numpy(w.v).cuda()
    res = {}
    if mode == "windows":
        owner = sharding.lpt_assign(sharding.window_costs(w.windows, points=w.points), world)
        op = anova_fast_operator(Dataset(w.points), spec, fit_fraction=w.fit_fraction,
                                 window_mask=sharding.window_mask(owner, rank))
        y = torch.empty_like(v)
        sharding.pipelined_matvec(op, v, y, 4, allreduce_async)
        res["pipelined"] = y.cpu().numpy()
        y2 = torch.empty_like(v)
        op.apply_into(v, y2)  # plain: one apply, one all-reduce
        allreduce(y2)
        res["plain"] = y2.cpu().numpy()
        part = torch.empty_like(v)
        op.apply_into(v, part)
        y3 = torch.empty_like(v)
        op.apply_windows(v)
        op.combine_range(y3, 0, w.n)
        res["combine_equals_apply"] = np.array([float(torch.equal(part, y3))])
    else:
        own = sharding.point_block(w.n, world, rank)
        op = sharding.PointShardedOperator(Dataset(w.points), spec, own, fit_fraction=w.fit_fraction)
        b = -(-w.n // world)
        y_pad = torch.zeros(world * b, dtype=torch.float64, device="cuda")
        op.matvec_blocks(v, y_pad, rank, world, allreduce, allgather)
        res["blocks"] = y_pad[:w.n].cpu().numpy()
        y = torch.empty_like(v)
        op.matvec(v, y, allreduce)
        res["allreduce"] = y.cpu().numpy()
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    dist.barrier()
    dist.destroy_process_group()


def _run(tmp_path, mode, case, world=2):
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_worker, args=(world, port, str(tmp_path), mode, case), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(world)]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _reference(oracle_lib, case):
    from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator
    cfg, n = CASES[case]
    w = workloads.make(cfg, n)
    single = anova_fast_operator(Dataset(w.points), AnovaKernelSpec(FeatureWindowing.explicit(w.windows)),
                                 fit_fraction=w.fit_fraction).apply(w.v)
    ref = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)
    return single, ref


@pytest.mark.parametrize("case", ["cfg3", "cfg5"])
def test_window_sharded_two_ranks(tmp_path, oracle_lib, case):
    out = _run(tmp_path, "windows", case)
    single, ref = _reference(oracle_lib, case)
    for r in out:
        for key in ("pipelined", "plain"):
            assert rel(r[key], single) <= 1e-12, key
            assert rel(r[key], ref) <= 1e-10, key
        assert np.array_equal(r["pipelined"], r["plain"])  # chunked sum == one all-reduce
        assert r["combine_equals_apply"][0] == 1.0
    assert np.array_equal(out[0]["pipelined"], out[1]["pipelined"])


@pytest.mark.parametrize("case", ["cfg2", "cfg5"])
def test_point_sharded_two_ranks(tmp_path, oracle_lib, case):
    out = _run(tmp_path, "points", case)
    single, ref = _reference(oracle_lib, case)
    for r in out:
        for key in ("blocks", "allreduce"):
            assert rel(r[key], single) <= 1e-12, key
            assert rel(r[key], ref) <= 1e-10, key
        assert np.array_equal(r["blocks"], r["allreduce"])  # y rows come from one owner either way


def test_pipelined_entry_points_check_their_arguments():
    """ksvm_nfft_op_apply_windows / _combine_range take device pointers and a
    window-sharded (not point-sharded) operator; the grid pool belongs to
    point-sharded operators; errors map to status 4 (std::invalid_argument)."""
    import torch
    from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, sharding
    w = workloads.make(2, 4000)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    op = anova_fast_operator(Dataset(w.points), spec)
    v = torch.from_numpy(w.v).cuda()
    y = torch.zeros_like(v)
    with pytest.raises(ValueError):
        op.apply_windows(w.v)  # host array
    op.apply_windows(v)
    for lo, hi in ((-1, 10), (0, w.n + 1), (20, 10)):
        with pytest.raises(ValueError):
            op.combine_range(y, lo, hi)
    op.combine_range(y, 0, 0)  # empty range: no-op
    assert float(y.abs().sum()) == 0.0
    pts = sharding.PointShardedOperator(Dataset(w.points), spec, sharding.point_block(w.n, 2, 0))
    assert pts.grid_pool().numel() == sum(g.numel() for g in pts.grids())


def test_point_shards_in_fp32_mode(oracle_lib):
    """fp32 mode on point-sharded operators: the shards' partial grids add up
    to the full product within the fp32 contract (1e-5)."""
    import torch
    from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, sharding
    w = workloads.make(5, 200000)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    shards = [sharding.PointShardedOperator(Dataset(w.points), spec, sharding.point_block(w.n, 2, r),
                                            fit_fraction=w.fit_fraction, precision="fp32") for r in range(2)]
    v = torch.from_numpy(w.v).cuda()
    for op in shards:
        op.apply_spread(v)
    pools = [op.grid_pool() for op in shards]
    total = pools[0] + pools[1]
    for p in pools:
        p.copy_(total)
    y = torch.zeros_like(v)
    for op in shards:
        part = torch.empty_like(v)
        op.apply_finish(part)
        y += part
    ref = oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)
    assert rel(y.cpu().numpy(), ref) <= 1e-5
