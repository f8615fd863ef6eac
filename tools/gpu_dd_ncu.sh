#!/bin/bash
# ncu --set full of the counting chain's kernels on config 4 (one resident step after warm-up).
mkdir -p gpurun_out
TAG=${1:-a}
timeout 600 python tools/dd_check.py 4 > gpurun_out/dd_check4_${TAG}.txt 2>&1; head -3 gpurun_out/dd_check4_${TAG}.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dd_aggregate|dd_expand_dev|dd_tile_sort|dd_rank" -s 8 -c 4 \
   -o gpurun_out/dd_ncu_${TAG} python tools/run_resident.py 4 3 > gpurun_out/dd_ncu_${TAG}.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/dd_ncu_${TAG}.log
