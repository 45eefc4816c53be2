timeout 400 python bench.py > gpurun_out/b24.log 2>&1; tail -1 gpurun_out/b24.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["phase_ms"], d["clocks"], d["roofline"]["frac"], d["roofline_gather"]["frac"])'
nvidia-smi --query-gpu=power.limit,power.default_limit,power.max_limit,enforced.power.limit --format=csv
