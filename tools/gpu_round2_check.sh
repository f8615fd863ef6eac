set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 compute-sanitizer --tool memcheck python -c "import torch; x=torch.ones(10,device='cuda'); print(x.sum())" > gpurun_out/cs_probe.log 2>&1; echo "cs rc=$?"; tail -5 gpurun_out/cs_probe.log
