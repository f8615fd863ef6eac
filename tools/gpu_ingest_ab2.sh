#!/bin/bash
# A/B of ingest builds (default = WS_I7_MINB 6) + ncu of the default ingest7.
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/ab_${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_${TAG}_tests.log
timeout 900 python tools/ab_quick.py "$@" > gpurun_out/ab_${TAG}.txt 2>&1; echo "ab rc=$?"
python - gpurun_out/ab_${TAG}.txt <<'PY'
import sys, json, re
for l in open(sys.argv[1]):
    m = re.match(r'\[(\d)\] (\S+)\s+(\{.*\})', l)
    if m:
        d = json.loads(m.group(3)); print(m.group(1), m.group(2), 'step', round(d['ms'],4), 'ingest', d['phases'].get('ingest'), 'radix_l0', d['phases'].get('radix_l0'))
    else: print(l.strip()[:300])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ingest" -s 14 -c 1 \
    -o gpurun_out/ncu_ingest_7_$TAG python tools/run_resident.py 4 2 > gpurun_out/ncu_ingest_7_$TAG.log 2>&1
echo "ncu rc=$?"
