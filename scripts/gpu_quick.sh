#!/bin/bash
# Quick check: GPU parity subset + config 5 / config 2 bench lines.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-quick}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
echo done
