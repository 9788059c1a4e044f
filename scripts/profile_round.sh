# Round profile: bench lines (configs 2, 4, 5), reference arm, ncu launch list and
# one full ncu capture. Outputs under gpurun_out/ (copied to profiles/ afterwards).
set -x
make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_cfg2.json 2> gpurun_out/ref_cfg2.err
python bench.py --config 4 --steps 50 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
# launch list: same command (config 2) with fewer steps, plain run first
ARGS="--steps 5 --warmup 3 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
ARGS4="--config 4 --steps 3 --warmup 3 --no-cpu-baseline"
python bench.py $ARGS4 > gpurun_out/plain_cfg4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"spread3|gather3|conv_stage|reduce" -s 8 -c 6 -o gpurun_out/prof_cfg4 python bench.py $ARGS4 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
