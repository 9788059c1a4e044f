#!/bin/bash
# 3xTF32 kernels with bounded accumulation chains: parity incl. full size, error, bench (4 vs 5 CTAs/SM spread), ncu.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2n; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests_t32.log 2>&1; echo "rc=$?" >> $O/tests_t32.log
timeout 1200 python -m pytest tests/test_gpu_fullsize_parity.py -q -x -p no:cacheprovider > $O/tests_full.log 2>&1; echo "rc=$?" >> $O/tests_full.log
timeout 600 python scripts/fp32_error.py > $O/error_tf32.jsonl 2> $O/error_tf32.err
for occ in 4 5; do
  KSVM_NFFT_T32OCC=$occ timeout 300 python bench.py --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_occ$occ.json 2> $O/bench5_occ$occ.err
done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 300 ncu --metrics $M --clock-control none -k regex:"t32_kernel" -c 2 --csv python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu5_t32.csv 2> $O/ncu5_t32.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"gather3_t32" -c 1 -f -o $O/gather3_t32 python bench.py --precision fp32 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_g.log 2>&1
echo done
