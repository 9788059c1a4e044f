#!/bin/bash
# Re-entry check: full GPU suite, config-5 / config-2 bench lines, source-level ncu of the d=3 kernels.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2c; mkdir -p $O
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
for K in spread3_s8 gather3_s8; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -f -o $O/$K \
  python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$K.log 2>&1
done
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
echo done
