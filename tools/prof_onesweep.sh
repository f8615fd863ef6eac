mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"radix_onesweep" -c 4 \
    -o gpurun_out/ncu_onesweep_r02 python tools/run_resident.py 4 1 > gpurun_out/ncu_onesweep_r02.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_onesweep_r02.log
