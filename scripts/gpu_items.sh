#!/bin/bash
# A/B of the d = 3 item sizing (items per SM) on config 5, plus the d = 1 kernels' launch times.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-items}; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for s in 24 36 48; do for g in 48 96; do
  KSVM_NFFT_ITEMS_PER_SM=$s KSVM_NFFT_GITEMS_PER_SM=$g timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/b5_${s}_${g}.json 2> $O/b5_${s}_${g}.err
done; done
echo done
