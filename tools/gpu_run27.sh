timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hot.py tests/test_gpu_fused.py -x -q > gpurun_out/pt27.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pt27.log
python tools/quick_sched.py c2,c3,c4,c5 merge_path
timeout 400 python bench.py --no-extras --steps 300 > gpurun_out/b27.log 2>&1; tail -1 gpurun_out/b27.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["phase_ms"])'
