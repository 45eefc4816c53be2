timeout 900 python -m pytest tests/test_gpu_sssp.py -x -q > gpurun_out/pt23.log 2>&1; echo "sssp tests rc=$?"; tail -3 gpurun_out/pt23.log
timeout 900 python tools/bench_sssp.py 20,22,24 > gpurun_out/sssp23.jsonl 2>&1; echo "bench rc=$?"; cat gpurun_out/sssp23.jsonl
