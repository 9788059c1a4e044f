#!/bin/bash
# A/B of the d = 3 item floors (spread KSVM_NFFT_ITEM3, gather KSVM_NFFT_GITEM) on configs 3 and 2.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-items3}; mkdir -p $O
export KSVM_NFFT_QUIET=1
for s in 1024 768 512 384; do for g in 512 256 128; do
  KSVM_NFFT_ITEM3=$s KSVM_NFFT_GITEM=$g timeout 300 python bench.py --config 3 --steps 100 --warmup 10 --no-cpu-baseline > $O/b3_${s}_${g}.json 2>/dev/null
done; done
for s in 1024 512; do for g in 512 128; do
  KSVM_NFFT_ITEM3=$s KSVM_NFFT_GITEM=$g timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/b2_${s}_${g}.json 2>/dev/null
done; done
echo done
