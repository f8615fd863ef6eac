#!/bin/bash
# A/B of radix builds on the resident step + tests + per-pass ncu of the default build.
TAG=${1:-x}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -m gpu -x -q > gpurun_out/ab_${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_${TAG}_tests.log
timeout 900 python tools/ab_quick.py "$@" > gpurun_out/ab_${TAG}.txt 2>&1; echo "ab rc=$?"
python - gpurun_out/ab_${TAG}.txt <<'PY'
import sys, json, re
for l in open(sys.argv[1]):
    m = re.match(r'\[(\d)\] (\S+)\s+(\{.*\})', l)
    if m:
        d = json.loads(m.group(3)); print(m.group(1), m.group(2), 'step', round(d['ms'],4), 'ingest', d['phases'].get('ingest'), 'radix_l0', d['phases'].get('radix_l0'), 'hist', d['phases'].get('radix_hist_l0'))
    else: print(l.strip()[:300])
PY
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"radix_onesweep" -c 4 --csv \
    --log-file gpurun_out/ncu_os_${TAG}.csv python tools/run_resident.py 4 1 > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launch_table.py gpurun_out/ncu_os_${TAG}.csv
