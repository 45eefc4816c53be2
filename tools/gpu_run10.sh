timeout 1200 python -m pytest tests/test_gpu_sssp.py -x -q > gpurun_out/pytest_sssp.log 2>&1; echo "pytest sssp rc=$?"; tail -15 gpurun_out/pytest_sssp.log
timeout 600 python tools/bench_sssp.py 20,22,24 > gpurun_out/bench_sssp.jsonl 2>&1; echo "bench sssp rc=$?"; cat gpurun_out/bench_sssp.jsonl | tail -12
