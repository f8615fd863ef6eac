#!/bin/bash
# ncu captures of the payload-mode ingest on the device-resident config-4 step
# (the launch inside ws_sort_resident, after the 14 chunked launches of the
# setup ingest): default (word-parallel ingest6) and WSORT_INGEST_V1=1.
# usage (GPU box): bash tools/prof_ingest.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:ingest6 -s 14 -c 1 \
    -o gpurun_out/ingest6_$TAG python tools/run_resident.py 4 2 > gpurun_out/ncu_ingest6_$TAG.log 2>&1
echo "ingest6 ncu rc=$?"
if [ "${2:-}" = v1 ]; then
WSORT_INGEST_V1=1 ncu --set full --clock-control none --import-source on -k regex:reserve_ingest -s 14 -c 1 \
    -o gpurun_out/ingest_v1_$TAG python tools/run_resident.py 4 2 > gpurun_out/ncu_ingest_v1_$TAG.log 2>&1
echo "v1 ncu rc=$?"
fi
