# warm-cache launch list (ncu --cache-control none) of a short bench run
make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
ARGS="--config ${CFG:-2} --steps 5 --warmup 3 --no-cpu-baseline ${EXTRA}"
python bench.py $ARGS > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_${TAG:-x}.csv python bench.py $ARGS > gpurun_out/ncu_l.log 2>&1
python scripts/launch_table.py gpurun_out/launches_${TAG:-x}.csv
