# Round profile: bench lines (configs 2..5), reference arm, warm ncu launch list (cfg2) and
# full ncu captures of the dominant kernels (cfg2 and cfg4). Outputs under gpurun_out/.
set -x
make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_cfg2.json 2> gpurun_out/ref_cfg2.err
python bench.py --config 3 --steps 100 --warmup 5 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --config 4 --steps 50 --warmup 5 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --config 5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
ARGS="--steps 5 --warmup 3 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_cfg2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
python bench.py $ARGS > gpurun_out/plain_cfg2b.log 2>&1 && \
ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -s 4 -c 2 -o gpurun_out/prof_cfg2 python bench.py $ARGS > gpurun_out/ncu_full2.log 2>&1
ARGS4="--config 4 --steps 3 --warmup 3 --no-cpu-baseline"
python bench.py $ARGS4 > gpurun_out/plain_cfg4.log 2>&1 && \
ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -s 4 -c 2 -o gpurun_out/prof_cfg4 python bench.py $ARGS4 > gpurun_out/ncu_full4.log 2>&1
python scripts/traffic.py cfg2=gpurun_out/prof_cfg2.ncu-rep cfg4=gpurun_out/prof_cfg4.ncu-rep > gpurun_out/traffic.json
python scripts/ncu_summary.py gpurun_out/prof_cfg2.ncu-rep > gpurun_out/ncu_cfg2_full.txt
python scripts/ncu_summary.py gpurun_out/prof_cfg4.ncu-rep > gpurun_out/ncu_cfg4_full.txt
python scripts/launch_table.py gpurun_out/launches_cfg2.csv > gpurun_out/launches_cfg2.txt
tail -1 gpurun_out/ncu_full2.log gpurun_out/ncu_full4.log
# end-to-end training and the callers of the matvec
python scripts/bench_ipm.py --config 1 --oracle > gpurun_out/ipm1.json 2>/dev/null
python scripts/bench_ipm.py --config 3 > gpurun_out/ipm3.json 2>/dev/null
python scripts/bench_ipm.py --config 5 > gpurun_out/ipm5.json 2>/dev/null
python scripts/bench_saddle.py > gpurun_out/saddle2.json 2>/dev/null
python scripts/bench_lowrank.py > gpurun_out/lowrank3.json 2>/dev/null
python scripts/bench_predict.py > gpurun_out/predict3.json 2>/dev/null
python scripts/bench_batch.py > gpurun_out/batch2.json 2>/dev/null
