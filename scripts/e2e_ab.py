"""A/B of the host-pointer apply (config 2): wall time per call through the
public API with pinned numpy views, as bench.py's e2e measures it."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2312_00538_b200 import AnovaKernelSpec, Dataset, FeatureWindowing, anova_fast_operator, workloads  # noqa: E402

w = workloads.make(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
op = anova_fast_operator(Dataset(w.points), AnovaKernelSpec(FeatureWindowing.explicit(w.windows)), fit_fraction=w.fit_fraction)
vh = torch.from_numpy(w.v).pin_memory()
yh = torch.empty_like(vh).pin_memory()
vn, yn = vh.numpy(), yh.numpy()
for _ in range(20):
    op.apply(vn, out=yn)
ts = []
for rep in range(5):
    t0 = time.perf_counter()
    for _ in range(200):
        op.apply(vn, out=yn)
    ts.append((time.perf_counter() - t0) / 200 * 1e6)
print(os.environ.get("KSVM_NFFT_HOSTGRAPH", "1"), "us/call", " ".join(f"{t:.1f}" for t in ts), "min %.1f" % min(ts))
