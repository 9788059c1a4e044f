#!/bin/bash
# Sliced tile_reduce: bench configs 3, 4, 5; launch lists of configs 3 and 4; parity subset.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2k; mkdir -p $O
timeout 300 python bench.py --config 3 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench3.json 2> $O/bench3.err
timeout 300 python bench.py --config 4 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench4.json 2> $O/bench4.err
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
for c in 3 4; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $O/launches_cfg$c.csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/ncu_l$c.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullsize_parity.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
echo done
