cd $GRAFT_REPO_ROOT; O=gpurun_out/f32c; mkdir -p $O
./scripts/micro/ffma_rates > $O/ffma_rates.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python bench.py --config 2 --precision fp32 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2_f32.json 2> $O/bench2_f32.err
