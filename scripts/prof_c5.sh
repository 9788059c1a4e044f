set -x
make -C paper_2312_00538_b200/csrc >/dev/null
mkdir -p gpurun_out
python bench.py --config 5 --n 2000000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p5.json 2>gpurun_out/p5.err && \
ncu --set full --clock-control none --import-source on -k regex:"spread3|gather3" -s 2 -c 2 -o gpurun_out/prof_c5 python bench.py --config 5 --n 2000000 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1
tail -5 gpurun_out/ncu_c5.log
python bench.py --steps 50 --warmup 5 > gpurun_out/b2.json 2> gpurun_out/b2.err; cat gpurun_out/b2.json
