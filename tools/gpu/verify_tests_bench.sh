nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r2_pt1.log 2>&1; echo "gpu tests rc=$?"; tail -30 gpurun_out/r2_pt1.log
timeout 600 python bench.py > gpurun_out/r2_bench1.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2_bench1.log
