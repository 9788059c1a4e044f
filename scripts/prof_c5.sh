# ncu capture of the 3D spread/gather kernels on config 5 (n=2M)
make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
ARGS="--config 5 --n 2000000 --steps 3 --warmup 3 --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/p5.json 2>gpurun_out/p5.err && \
ncu --set full --clock-control none --import-source on -k regex:"spread3|gather3" -s 2 -c 2 -o gpurun_out/prof_c5_${TAG:-x} python bench.py $ARGS > gpurun_out/ncu_c5.log 2>&1
tail -2 gpurun_out/ncu_c5.log
