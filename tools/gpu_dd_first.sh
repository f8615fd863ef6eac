#!/bin/bash
# Distinct-word counting path: parity on configs 1-4, its tests, A/B against the sort paths.
mkdir -p gpurun_out
for c in 1 2 3; do timeout 300 python tools/dd_check.py $c > gpurun_out/dd_check$c.txt 2>&1; head -2 gpurun_out/dd_check$c.txt; done
timeout 600 python tools/dd_check.py 4 > gpurun_out/dd_check4.txt 2>&1; head -30 gpurun_out/dd_check4.txt
timeout 900 python -m pytest tests/test_gpu_counting.py -x -q 2>&1 | tail -15 > gpurun_out/dd_tests.txt; cat gpurun_out/dd_tests.txt
timeout 600 python tools/ab_quick.py default env:WSORT_NO_DEDUPE=1 > gpurun_out/dd_ab.txt 2>&1; cut -c1-420 gpurun_out/dd_ab.txt
