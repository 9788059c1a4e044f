#!/bin/bash
# fp32 mode: 3xTF32 tensor-core kernels vs the FFMA kernels (parity, config-5 bench, error, ncu metrics).
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2m; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests_t32.log 2>&1; echo "rc=$?" >> $O/tests_t32.log
KSVM_NFFT_F32K=ffma timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests_ffma.log 2>&1; echo "rc=$?" >> $O/tests_ffma.log
for k in tf32 ffma; do
  KSVM_NFFT_F32K=$k timeout 300 python bench.py --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_$k.json 2> $O/bench5_$k.err
  KSVM_NFFT_F32K=$k timeout 600 python scripts/fp32_error.py > $O/error_$k.jsonl 2> $O/error_$k.err
done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:"t32_kernel" -c 2 --csv python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu5_t32.csv 2> $O/ncu5_t32.err
echo done
