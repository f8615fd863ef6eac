#!/bin/bash
# Correctness evidence on the current code: GPU suite (shipped build, then the
# checked build with device bounds checks), randomised stress (default knobs,
# then counting from the smallest text with the small-corpus kernel off),
# dirty-memory repeats, repeated config-4 parity of the counting path.
TAG=${1:-x}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/ev_${TAG}_suite.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/ev_${TAG}_suite.log
WSORT_LIB=$PWD/build/checked/libwsort_b200.so WSORT_CHECKED=1 timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/ev_${TAG}_checked.log 2>&1; echo "checked suite rc=$?"; tail -2 gpurun_out/ev_${TAG}_checked.log
timeout 500 python tools/stress.py ${STRESS_S:-300} ${SEED:-11} > gpurun_out/ev_${TAG}_stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/ev_${TAG}_stress.log
WSORT_DEDUPE_MIN=0 WSORT_NO_TINY=1 timeout 500 python tools/stress.py ${STRESS_S:-300} ${SEED:-12} > gpurun_out/ev_${TAG}_stress_counting.log 2>&1; echo "stress (counting everywhere) rc=$?"; tail -3 gpurun_out/ev_${TAG}_stress_counting.log
timeout 600 python tools/flaky2.py > gpurun_out/ev_${TAG}_flaky2.log 2>&1; echo "flaky2 rc=$?"; tail -2 gpurun_out/ev_${TAG}_flaky2.log
for i in 1 2 3 4 5 6; do timeout 300 python tools/dd_check.py 4 2>/dev/null | head -1; done > gpurun_out/ev_${TAG}_dd_repeat.log; cat gpurun_out/ev_${TAG}_dd_repeat.log
