#!/bin/bash
# Source-level ncu capture of one kernel (regex $2) at config $3 (default 5).
TAG=${1:-src}; K=${2:-gather3_s8}; CFG=${3:-5}
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$TAG
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$K" -c 1 -f -o gpurun_out/$TAG/k \
  python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/ncu.log 2>&1
echo done
