#!/bin/bash
# ncu --set full of the counting chain's kernels on config 4 (one resident step after warm-up).
mkdir -p gpurun_out
TAG=${1:-a}
KERN=${2:-dd_aggregate|dd_expand_dev|dd_tile_sort|dd_rank}
N=${3:-4}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KERN" -s $((2*N)) -c $N \
   -o gpurun_out/dd_ncu_${TAG} python tools/run_resident.py 4 3 > gpurun_out/dd_ncu_${TAG}.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/dd_ncu_${TAG}.log
