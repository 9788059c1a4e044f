#!/bin/bash
# A/B: item order (LPT), spread batch 16/32, gather 5 CTAs/SM; config 5 and 3 bench lines each.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2e; mkdir -p $O
run() { # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_$tag.json 2> $O/bench5_$tag.err
  env "$@" timeout 300 python bench.py --config 3 --steps 50 --warmup 10 --no-cpu-baseline > $O/bench3_$tag.json 2> $O/bench3_$tag.err
}
run base KSVM_NFFT_LPT=0
run lpt KSVM_NFFT_LPT=1
run lpt_b16 KSVM_NFFT_LPT=1 KSVM_NFFT_S3B=16
run lpt_g5 KSVM_NFFT_LPT=1 KSVM_NFFT_G3OCC=5
run lpt_b16_g5 KSVM_NFFT_LPT=1 KSVM_NFFT_S3B=16 KSVM_NFFT_G3OCC=5
timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
timeout 300 python bench.py --config 4 --steps 50 --warmup 10 --no-cpu-baseline > $O/bench4.json 2> $O/bench4.err
KSVM_NFFT_S3B=16 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_fullsize_parity.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
echo done
