#!/bin/bash
# Quick build-measure loop on the GPU box: parity subset, config-5 and
# config-2 bench lines, and a compact ncu metric set for the d=3 kernels.
#   gpurun -- 'bash scripts/gpu_iter.sh TAG'
TAG=${1:-iter}
cd $GRAFT_REPO_ROOT
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_properties.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench5.json 2> $O/bench5.err
timeout 300 python bench.py --config 2 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum
timeout 300 ncu --metrics $M --clock-control none -k regex:"spread3_s8|gather3_s8|spread3c|gather3c" -c 4 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu5.csv 2> $O/ncu5.err
timeout 300 ncu --metrics $M --clock-control none -k regex:"spread3|gather3" -c 4 --csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu2.csv 2> $O/ncu2.err
echo done
