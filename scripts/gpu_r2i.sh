#!/bin/bash
# Micro: fenced (clumped) DMULs; A/B of KSVM_NFFT_CLUMP on config 5; parity under CLUMP=1.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2i; mkdir -p $O
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_interleave scripts/micro/dmma_interleave.cu 2>/dev/null && /tmp/dmma_interleave > $O/micro_interleave.txt 2>&1
bash scripts/gpu_ab.sh r2i KSVM_NFFT_CLUMP=0,1
echo done
