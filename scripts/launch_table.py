"""Per-kernel mean/min durations from an ncu --metrics gpu__time_duration.sum CSV."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.OrderedDict()
for r in data:
    name = r[ki].split("(")[0].replace("void ", "").replace("ksvm_nfft::", "")[:44]
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0))
for k, v in agg.items():
    print(f"{k:46s} n={len(v):4d} mean={sum(v)/len(v):9.2f} us  min={min(v):9.2f} us")
