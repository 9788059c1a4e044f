"""Diagnostic: where a small (config 2) apply's time goes. Prints the
bench-style step time (256 MiB L2 flush before each step), warm single-apply
latency, back-to-back throughput, and the floor of one trivial kernel between
the same two events. Run under env variants (KSVM_NFFT_NO_GRAPH=1,
KSVM_NFFT_PDL=0, ...) in separate processes."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, workloads

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = workloads.make(cfg)
op = anova_fast_operator(Dataset(w.points), AnovaKernelSpec(FeatureWindowing.explicit(w.windows)),
                         fit_fraction=w.fit_fraction)
v = torch.from_numpy(w.v).cuda()
y = torch.empty_like(v)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
tiny = torch.empty(8, device="cuda")
for _ in range(10):
    op.apply_into(v, y)
torch.cuda.synchronize()
out = {}
K = 100
for mode in ("flush", "warm", "trivial", "back2back"):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    if mode == "back2back":
        a, b = ev[0]
        a.record()
        for k in range(K):
            op.apply_into(v, y)
        b.record()
        torch.cuda.synchronize()
        out[mode] = a.elapsed_time(b) / K * 1e3
        continue
    for k in range(K):
        if mode == "flush":
            flush.zero_()
        else:
            torch.cuda._sleep(300000)  # keep the host ahead of the GPU
        ev[k][0].record()
        if mode == "trivial":
            tiny.zero_()
        else:
            op.apply_into(v, y)
        ev[k][1].record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    out[mode] = ts[K // 2]
tag = " ".join(f"{k}={os.environ[k]}" for k in sorted(os.environ) if k.startswith("KSVM_NFFT_")) or "default"
print(f"cfg{cfg} [{tag}] " + "  ".join(f"{k} {v:7.1f} us" for k, v in out.items()), flush=True)
