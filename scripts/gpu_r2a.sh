cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_tests.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench5.json 2> gpurun_out/r2a_bench5.err
timeout 300 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_bench2.json 2> gpurun_out/r2a_bench2.err
timeout 400 ncu --set full --import-source on --clock-control none -k regex:"spread3_s8|gather3_s8" -c 2 -f -o gpurun_out/r2a_cfg5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2a_launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_ncu2.log 2>&1
echo done
