#!/bin/bash
# A/B: per-cell (split-power) vs column d=3 kernels at the sparse configs 2 and 3; config 5 with the wide tile_reduce.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2g; mkdir -p $O
for c in 2 3; do
 for s in column cell; do for g in column cell; do
  KSVM_NFFT_SPREAD3=$s KSVM_NFFT_GATHER3=$g timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > $O/bench${c}_s${s}_g${g}.json 2> $O/bench${c}_s${s}_g${g}.err
 done; done
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
timeout 300 python bench.py --config 4 --steps 50 --warmup 10 --no-cpu-baseline > $O/bench4.json 2> $O/bench4.err
echo done
