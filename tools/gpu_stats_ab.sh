#!/bin/bash
# Stats-mode A/B of library builds (+ parity tests of the default build).
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/st_${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/st_${TAG}_tests.log
AB_STATS=1 timeout 900 python tools/ab_quick.py "$@" > gpurun_out/st_${TAG}.txt 2>&1; echo "ab rc=$?"
python - gpurun_out/st_${TAG}.txt <<'PY'
import sys, json, re
for l in open(sys.argv[1]):
    m = re.match(r'\[(\d)\] (\S+)\s+(\{.*\})', l)
    if m:
        d = json.loads(m.group(3)); ph = d['phases']
        print(m.group(1), m.group(2), 'step', round(d['ms'],4), ' '.join(f"{k}={v}" for k, v in ph.items() if k.startswith(('merge', 'tile', 'ingest', 'reorder'))))
    else: print(l.strip()[:300])
PY
