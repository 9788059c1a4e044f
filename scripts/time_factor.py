"""Where config 3's Nystrom factor time goes: one-window operator creation
vs the sketch itself, per window."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_00538_b200 import (Dataset, balance_and_split, fast_window_operator, nystrom, workloads,  # noqa: E402
                                   zscore_fit_transform)

w = workloads.make(3)
tr, te = balance_and_split(Dataset(w.points, w.labels), 0.5, 0)
zscore_fit_transform(tr, te)
fast_window_operator(tr.points[:1000], w.windows[0], 1.0)  # warm-up
for l, win in enumerate(w.windows):
    t0 = time.perf_counter()
    fop = fast_window_operator(tr.points, win, 1.0)
    t1 = time.perf_counter()
    f = nystrom(fop, 25, "gaussian", l)
    t2 = time.perf_counter()
    print(f"window {l} d={len(win)}: create {1e3 * (t1 - t0):.1f} ms, nystrom {1e3 * (t2 - t1):.1f} ms")
