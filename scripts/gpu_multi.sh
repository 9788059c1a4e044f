#!/bin/bash
# Multi-rank paths on a 1-GPU lease: 2-rank GPU tests (gloo, ranks share
# cuda:0) and the torchrun bench in both shard modes; plus the parity subset.
TAG=${1:-multi}
cd $GRAFT_REPO_ROOT; O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_sharding.py tests/test_gpu_parity.py tests/test_gpu_lowrank.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for sh in windows points; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 5 --warmup 3 --shard $sh --backend gloo --same-device --config 5 > $O/bench5_2r_$sh.json 2> $O/bench5_2r_$sh.err
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
echo done
