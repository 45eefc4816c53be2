timeout 600 python -m pytest tests/test_gpu_hot.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest15.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest15.log
timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/b15.log 2>&1; tail -1 gpurun_out/b15.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"], d["roofline_gather"])'
