make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
ARGS="--config 2 --steps 3 --warmup 3 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/p2.json 2>gpurun_out/p2.err && \
ncu --set full --clock-control none --import-source on -k regex:"spread3|gather3|conv_stage|reduce|spread2|gather2" -s 9 -c 9 -o gpurun_out/prof_c2_${TAG:-x} python bench.py $ARGS > gpurun_out/ncu_c2.log 2>&1
tail -2 gpurun_out/ncu_c2.log
