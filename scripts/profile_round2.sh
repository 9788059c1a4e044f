#!/bin/bash
# Round-2 profile capture (run on the GPU box): bench lines, reference arm,
# warm launch lists, ncu --set full captures of the d = 3 kernels, training.
# Outputs under gpurun_out/r2p/; the summaries are copied into profiles/.
cd $GRAFT_REPO_ROOT; O=gpurun_out/r2p; mkdir -p $O
export KSVM_NFFT_QUIET=1
nproc > $O/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/host.txt; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv >> $O/host.txt
timeout 900 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_cfg5.json 2> $O/ref_cfg5.err
timeout 600 python bench.py --precision fp32 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_cfg5_fp32.json 2> $O/bench_cfg5_fp32.err
timeout 600 python bench.py --config 2 --steps 100 --warmup 10 > $O/bench_cfg2.json 2> $O/bench_cfg2.err
timeout 600 python bench.py --config 3 --steps 100 --warmup 10 > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 600 python bench.py --config 4 --steps 50 --warmup 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err
A5="--steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $O/launches_cfg5.csv python bench.py $A5 > $O/ncu_l5.log 2>&1
A2="--config 2 --steps 5 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 400 --csv --log-file $O/launches_cfg2.csv python bench.py $A2 > $O/ncu_l2.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -c 2 -f -o $O/full_cfg5 python bench.py $A5 > $O/ncu_f5.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"f32_kernel|t32_kernel" -c 2 -f -o $O/full_cfg5_fp32 python bench.py --precision fp32 $A5 > $O/ncu_f5b.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -s 4 -c 2 -f -o $O/full_cfg2 python bench.py $A2 > $O/ncu_f2.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -s 4 -c 2 -f -o $O/full_cfg3 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_f3.log 2>&1
timeout 600 ncu --set full --clock-control none --cache-control all --import-source on -k regex:"spread3|gather3" -s 4 -c 2 -f -o $O/full_cfg4 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_f4.log 2>&1
timeout 600 python scripts/bench_ipm.py --config 1 --oracle > $O/ipm1.json 2> $O/ipm1.err
timeout 600 python scripts/bench_ipm.py --config 3 > $O/ipm3.json 2> $O/ipm3.err
timeout 900 python scripts/bench_ipm.py --config 5 > $O/ipm5.json 2> $O/ipm5.err
timeout 1500 python scripts/ipm_scaling.py > $O/ipm_scaling.jsonl 2> $O/ipm_scaling.err
timeout 600 python scripts/fp32_error.py > $O/precision_error.jsonl 2> $O/precision_error.err
for m in dmma_interleave mma_legacy_rates; do nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/$m scripts/micro/$m.cu 2>/dev/null && /tmp/$m > $O/micro_$m.txt 2>&1; done
echo done
