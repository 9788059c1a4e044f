"""Histogram of executed SASS opcodes (per warp) + stall samples from an ncu source page CSV."""
import collections
import csv
import sys

r = list(csv.reader(sys.stdin))
h = next(x for x in r if 'Instructions Executed' in x)
ie, src, smp = h.index('Instructions Executed'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
warps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
op, st, tot, ts = collections.Counter(), collections.Counter(), 0, 0
for x in r:
    if len(x) != len(h) or not x[ie].isdigit():
        continue
    parts = x[src].split()
    if not parts:
        continue
    o = (parts[1] if parts[0].startswith('@') else parts[0]).split('.')[0]
    n, s = int(x[ie]), int(x[smp] or 0)
    op[o] += n; st[o] += s; tot += n; ts += s
print('instructions per warp', tot / warps, 'samples', ts)
for o, n in op.most_common(32):
    print(f'{o:10s} {n / warps:9.1f} {st[o] / max(ts, 1) * 100:5.1f}%')
