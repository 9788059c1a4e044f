"""GPU: point sharding (SURVEY.md 8(e) hybrid) on one device. The ranks'
shares are built as separate operators in one process and their partial
grids are summed in between (what the per-window NCCL all-reduce does across
GPUs); the sum of the shards' outputs must equal the unsharded operator and
the oracle. No rank waits on another: the phases run one after the other."""
import numpy as np
import pytest
import torch

import oracle
from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, workloads
from paper_2312_00538_b200.sharding import PointShardedOperator, point_shard

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("cfg,n,world", [(2, 20000, 2), (3, 12000, 3), (1, 2000, 4), (5, 30000, 2)])
def test_point_shards_sum_to_the_operator(oracle_lib, cfg, n, world):
    w = workloads.make(cfg, n)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    shards = [PointShardedOperator(Dataset(w.points), spec, point_shard(w.n, world, r), fit_fraction=w.fit_fraction)
              for r in range(world)]
    v = torch.from_numpy(w.v).cuda()
    for op in shards:
        op.apply_spread(v)
    grids = [op.grids() for op in shards]
    for k in range(len(grids[0])):  # the all-reduce of grid k
        total = sum(g[k] for g in grids)
        for g in grids:
            g[k].copy_(total)
    ys = []
    for op in shards:
        y = torch.empty_like(v)
        op.apply_finish(y)
        ys.append(y)
    y = sum(ys).cpu().numpy()
    full = anova_fast_operator(Dataset(w.points), spec, fit_fraction=w.fit_fraction).apply(w.v)
    assert rel(y, full) <= 1e-12
    assert rel(y, oracle_lib.anova(w.points, w.windows, fit=w.fit_fraction).apply(w.v)) <= 1e-10
    # each shard's output is zero off its own rows
    for r, yr in enumerate(ys):
        mask = np.ones(w.n, dtype=bool)
        mask[point_shard(w.n, world, r)] = False
        assert np.all(yr.cpu().numpy()[mask] == 0.0)


def test_point_shard_host_path_and_errors():
    w = workloads.make(2, 3000)
    spec = AnovaKernelSpec(FeatureWindowing.explicit(w.windows))
    op = PointShardedOperator(Dataset(w.points), spec, np.arange(w.n))
    op.apply_spread(w.v.copy())
    y = np.empty(w.n)
    op.apply_finish(y)
    full = anova_fast_operator(Dataset(w.points), spec).apply(w.v)
    assert rel(y, full) <= 1e-12
    for bad in ([], [5, 3], [-1, 2], [0, w.n]):
        with pytest.raises(ValueError):
            PointShardedOperator(Dataset(w.points), spec, np.asarray(bad, dtype=np.int64))
