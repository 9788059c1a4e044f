#!/bin/bash
# fp32 mode: parity tests, config-5 / config-2 bench lines in both precisions.
TAG=${1:-f32}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python bench.py --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_f32.json 2> $O/bench5_f32.err
timeout 300 python bench.py --config 2 --precision fp32 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2_f32.json 2> $O/bench2_f32.err
M=gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
timeout 300 ncu --metrics $M --clock-control none -k regex:"f32_kernel" -c 2 --csv python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu5.csv 2> $O/ncu5.err
echo done
