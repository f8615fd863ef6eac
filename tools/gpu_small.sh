#!/bin/bash
# Small-corpus path: GPU tests + configs 0-3 resident step with / without the tiny path.
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/small_${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/small_${TAG}_tests.log
timeout 600 python tools/small_configs.py 0 1 2 3 2>&1 | tail -4
WSORT_NO_TINY=1 timeout 600 python tools/small_configs.py 0 1 2>&1 | tail -2
