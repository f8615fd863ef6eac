python tools/resident_timeline.py 0 > gpurun_out/tl_c0.txt 2>&1; cat gpurun_out/tl_c0.txt
python tools/resident_timeline.py 1 > gpurun_out/tl_c1.txt 2>&1; cat gpurun_out/tl_c1.txt
WSORT_TRACE=2 python tools/run_resident.py 0 3 2>&1 | grep marks | tail -1
