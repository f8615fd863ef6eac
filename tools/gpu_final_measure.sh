#!/bin/bash
# Round-end measurement set: bench (config 4) + configs 0-3, the sort paths
# alone (WSORT_NO_DEDUPE=1), reference arm, timeline, launch list of the bench
# command. (ncu --set full captures: tools/gpu_dd_ncu.sh; their reports are
# large, keep gpurun_out/ under 64 MiB or nothing is copied back.)
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/fm_${TAG}_bench.json 2> gpurun_out/fm_${TAG}_bench.err; echo "bench rc=$?"
for c in 0 1 2 3; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/fm_${TAG}_bench_c$c.json 2> gpurun_out/fm_${TAG}_bench_c$c.err; echo "bench c$c rc=$?"
done
WSORT_NO_DEDUPE=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/fm_${TAG}_bench_sortpaths.json 2> gpurun_out/fm_${TAG}_bench_sortpaths.err; echo "bench (sort paths) rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fm_${TAG}_ref.json 2> gpurun_out/fm_${TAG}_ref.err; echo "ref rc=$?"
timeout 300 python tools/dd_check.py 4 > gpurun_out/fm_${TAG}_timeline_config4.txt 2>/dev/null; head -1 gpurun_out/fm_${TAG}_timeline_config4.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/fm_${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
