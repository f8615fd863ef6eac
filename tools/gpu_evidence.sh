#!/bin/bash
# Correctness evidence on the current code: GPU suite against the checked
# build (device bounds checks), randomised stress, dirty-memory repeats.
TAG=${1:-x}
mkdir -p gpurun_out
WSORT_LIB=$PWD/build/checked/libwsort_b200.so WSORT_CHECKED=1 timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/ev_${TAG}_checked.log 2>&1; echo "checked suite rc=$?"; tail -2 gpurun_out/ev_${TAG}_checked.log
timeout 900 python tools/stress.py 420 ${SEED:-11} > gpurun_out/ev_${TAG}_stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/ev_${TAG}_stress.log
timeout 600 python tools/flaky2.py > gpurun_out/ev_${TAG}_flaky2.log 2>&1; echo "flaky2 rc=$?"; tail -2 gpurun_out/ev_${TAG}_flaky2.log
