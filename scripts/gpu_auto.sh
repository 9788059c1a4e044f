#!/bin/bash
# bench.py --shard auto under torchrun, ranks sharing cuda:0 (gloo): 2 ranks -> windows, 4 -> points.
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-auto}; mkdir -p $O
export KSVM_NFFT_QUIET=1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --steps 3 --warmup 3 --backend gloo --same-device > $O/b5_$N.json 2> $O/b5_$N.err
done
echo done
