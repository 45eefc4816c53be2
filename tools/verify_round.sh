set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/v_gpu_tests.log
tail -3 gpurun_out/v_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.log 2>&1; tail -1 gpurun_out/v_bench.log
timeout 600 python bench.py --impl reference > gpurun_out/v_bench_ref.log 2>&1; tail -1 gpurun_out/v_bench_ref.log
