#!/bin/bash
# A/B of an env-selected kernel variant: bench config 5 and 2 under each
# setting of $2 (VAR=a,b), plus a compact ncu of the d=3 kernels.
TAG=${1:-ab}; VAR=${2%%=*}; VALS=${2#*=}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$TAG; mkdir -p $O
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for v in ${VALS//,/ }; do
  export $VAR=$v
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_$v.json 2> $O/bench5_$v.err
  timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2_$v.json 2> $O/bench2_$v.err
  timeout 300 ncu --metrics $M --clock-control none -k regex:"spread3|gather3" -c 2 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu5_$v.csv 2> $O/ncu5_$v.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
echo done
