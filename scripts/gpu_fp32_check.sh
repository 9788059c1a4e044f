#!/bin/bash
# fp32 mode check: parity, config-5 bench line, ncu metrics and source-level captures of the 3xTF32 kernels.
cd $GRAFT_REPO_ROOT; O=gpurun_out/fp32_check; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests_t32.log 2>&1; echo "rc=$?" >> $O/tests_t32.log
timeout 300 python bench.py --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 300 ncu --metrics $M --clock-control none -k regex:"t32_kernel" -c 2 --csv python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu5_t32.csv 2> $O/ncu5_t32.err
for K in spread3_t32 gather3_t32; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -f -o $O/$K python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$K.log 2>&1
done
echo done
