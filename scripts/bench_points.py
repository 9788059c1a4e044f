"""Point-sharded multi-GPU matvec timing (SURVEY.md 8(e) hybrid; the
default bench.py shards windows, as north_star prescribes):

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
      scripts/bench_points.py --config 5 --steps 20

Every rank owns a contiguous 1/N of the points of every window; one step is
spread (owned points) -> one NCCL all-reduce per window grid -> convolution,
gather (owned points), window sum -> one all-reduce of y. Same timing rules
as bench.py (L2 flush before each step, CUDA events, max over ranks). Prints
one JSON line on rank 0."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, workloads  # noqa: E402
from paper_2312_00538_b200.sharding import PointShardedOperator, point_shard  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--warmup", type=int, default=3)
a = ap.parse_args()
world, rank, local = (int(os.environ.get(k, d)) for k, d in (("WORLD_SIZE", "1"), ("RANK", "0"), ("LOCAL_RANK", "0")))
dev = torch.device("cuda", local)
torch.cuda.set_device(dev)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
os.environ.setdefault("KSVM_NFFT_QUIET", "1")
w = workloads.make(a.config, a.n)
op = PointShardedOperator(Dataset(w.points), AnovaKernelSpec(FeatureWindowing.explicit(w.windows)),
                          point_shard(w.n, world, rank), fit_fraction=w.fit_fraction, device=local)
v = torch.from_numpy(w.v).to(dev)
y = torch.empty_like(v)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
reduce = dist.all_reduce if world > 1 else None
for _ in range(max(3, a.warmup)):
    op.matvec(v, y, reduce)
torch.cuda.synchronize(dev)
if world > 1:
    dist.barrier()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
for k in range(a.steps):
    flush.zero_()
    ev[k][0].record()
    op.matvec(v, y, reduce)
    ev[k][1].record()
torch.cuda.synchronize(dev)
t = torch.tensor([sum(s.elapsed_time(e) for s, e in ev)], dtype=torch.float64, device=dev)
if world > 1:
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
ms = float(t.item()) / a.steps
if rank == 0:
    print(json.dumps({"metric": "ANOVA-NFFT kernel matvecs/sec (fp64)", "value": 1e3 / ms, "unit": "matvecs/s",
                      "n_gpus": world, "steps": a.steps, "ms_per_step": ms, "scaling": "strong",
                      "parallelism": f"point-sharded x{world}: per-window grid all-reduce + y all-reduce",
                      "config": {"workload": w.name, "n": w.n}}))
if world > 1:
    dist.destroy_process_group()
