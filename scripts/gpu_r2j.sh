#!/bin/bash
# Item-size sweep at the mid-size configs 3 and 4 (with largest-first dispatch) + the new order test.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "item_order or variants" > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for c in 3 4; do
 for i in 768 1024 1536 2048; do
  KSVM_NFFT_ITEM3=$i timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > $O/bench${c}_item$i.json 2> $O/bench${c}_item$i.err
 done
 for g in 256 384 512 768 1024; do
  KSVM_NFFT_GITEM=$g timeout 300 python bench.py --config $c --steps 100 --warmup 10 --no-cpu-baseline > $O/bench${c}_gitem$g.json 2> $O/bench${c}_gitem$g.err
 done
done
echo done
