# ncu full capture of kernels matching $K on bench --config $CFG
make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
ARGS="--config ${CFG:-2} --steps 3 --warmup 3 --no-cpu-baseline ${EXTRA}"
python bench.py $ARGS > gpurun_out/pk.json 2>gpurun_out/pk.err && \
ncu --set full --clock-control none --cache-control none --import-source on -k regex:"${K}" -s ${SKIP:-6} -c ${COUNT:-2} -o gpurun_out/prof_${TAG:-x} python bench.py $ARGS > gpurun_out/ncu_k.log 2>&1
tail -1 gpurun_out/ncu_k.log
