#!/bin/bash
# L2 eviction hints check: parity subset + reference-driver fixtures, config 5
# bench lines (fp64, fp32) and ncu --set full captures for DRAM traffic.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-r2b}; mkdir -p $O
export KSVM_NFFT_QUIET=1
timeout 1200 python -m pytest tests/test_gpu_ref_driver.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fp32.py tests/test_gpu_multirank.py -q -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
timeout 600 python bench.py --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_fp32.json 2> $O/bench5_fp32.err
A5="--steps 2 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -c 2 -f -o $O/full_cfg5 python bench.py $A5 > $O/ncu_f5.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"f32_kernel" -c 2 -f -o $O/full_cfg5_fp32 python bench.py --precision fp32 $A5 > $O/ncu_f5b.log 2>&1
echo done
