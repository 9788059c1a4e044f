"""Diagnostic: apply time with and without the 256 MiB L2 flush (config 2)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, workloads

w = workloads.make(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
op = anova_fast_operator(Dataset(w.points), AnovaKernelSpec(FeatureWindowing.explicit(w.windows)),
                         fit_fraction=w.fit_fraction)
v = torch.from_numpy(w.v).cuda()
y = torch.empty_like(v)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(5):
    op.apply_into(v, y)
torch.cuda.synchronize()
for mode in ("flush", "warm", "back2back"):
    K = 50
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if mode == "back2back":
        a, b = ev[0]
        a.record()
        for k in range(K):
            op.apply_into(v, y)
        b.record()
        torch.cuda.synchronize()
        print(f"{mode:10s} {a.elapsed_time(b) / K * 1e3:7.1f} us/apply")
        continue
    for k in range(K):
        if mode == "flush":
            flush.zero_()
        else:
            torch.cuda._sleep(200000)  # keep the queue ahead of the GPU
        ev[k][0].record()
        op.apply_into(v, y)
        ev[k][1].record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    print(f"{mode:10s} median {ts[K // 2]:7.1f} us  min {ts[0]:7.1f}")
