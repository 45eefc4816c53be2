LB_HOT_W=32 timeout 600 python -m pytest tests/test_gpu_hot.py -x -q > gpurun_out/pytest_lean.log 2>&1; echo "pytest lean rc=$?"; tail -3 gpurun_out/pytest_lean.log
for W in 16 32; do for L in 1016 504; do for slots in 16384 24576 32768 40960; do
  LB_HOT_W=$W timeout 300 python bench.py --no-extras --steps 100 --warmup 5 --items-per-tile $L --hot-slots $slots > gpurun_out/sw.log 2>&1
  echo "W $W L $L slots $slots: $(tail -1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["plan"]["hot_nnz_frac"], d["phase_ms"]["main"], d["roofline"]["kernel"])' 2>&1 | tail -1)"
done; done; done
