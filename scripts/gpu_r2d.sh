#!/bin/bash
# A/B of the split-power dense d=3 kernels + DMUL/DMMA interleave microbenchmark.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2d; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_interleave scripts/micro/dmma_interleave.cu && /tmp/dmma_interleave > $O/micro_interleave.txt 2>&1
bash scripts/gpu_ab.sh r2d KSVM_NFFT_D3=pair,split
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_properties.py -q -x -p no:cacheprovider > $O/tests_full.log 2>&1; echo "rc=$?" >> $O/tests_full.log
echo done
