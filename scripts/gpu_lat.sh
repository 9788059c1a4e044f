#!/bin/bash
cd $GRAFT_REPO_ROOT; O=gpurun_out/${1:-lat}; mkdir -p $O
export KSVM_NFFT_QUIET=1
( python scripts/latency.py 2
  KSVM_NFFT_NO_GRAPH=1 python scripts/latency.py 2
  KSVM_NFFT_PDL=0 python scripts/latency.py 2
  python scripts/latency.py 3
  python scripts/latency.py 1 ) > $O/lat.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv \
  python scripts/latency.py 2 > $O/launch_c2.csv 2> $O/launch_c2.err
echo done
