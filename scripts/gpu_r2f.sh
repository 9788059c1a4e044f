#!/bin/bash
# A/B of the spread item order (0: tile order, 1: largest first over the class, 2: per window) + full GPU suite.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2f; mkdir -p $O
for v in 0 1 2; do
  KSVM_NFFT_LPT=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5_lpt$v.json 2> $O/bench5_lpt$v.err
  KSVM_NFFT_LPT=$v timeout 300 python bench.py --config 3 --steps 50 --warmup 10 --no-cpu-baseline > $O/bench3_lpt$v.json 2> $O/bench3_lpt$v.err
  KSVM_NFFT_LPT=$v timeout 300 python bench.py --config 4 --steps 50 --warmup 10 --no-cpu-baseline > $O/bench4_lpt$v.json 2> $O/bench4_lpt$v.err
done
timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
echo done
