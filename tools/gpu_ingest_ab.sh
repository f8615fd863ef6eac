#!/bin/bash
# A/B + ncu of the payload-mode ingest variants (WSORT_INGEST=reserve|6|7).
# usage (GPU box): bash tools/gpu_ingest_ab.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/ab_${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_${TAG}_tests.log
timeout 600 python tools/ab_quick.py env:WSORT_INGEST=reserve env:WSORT_INGEST=7 > gpurun_out/ab_${TAG}.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/ab_${TAG}.txt | tail -30
for V in 7 reserve; do
WSORT_INGEST=$V timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ingest" -s 14 -c 1 \
    -o gpurun_out/ncu_ingest_${V}_$TAG python tools/run_resident.py 4 2 > gpurun_out/ncu_ingest_${V}_$TAG.log 2>&1
echo "ncu $V rc=$?"
done
