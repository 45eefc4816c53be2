python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_matrix.py c2,c3,c4,c5 > gpurun_out/landscape.jsonl 2> gpurun_out/landscape.err; echo "landscape rc=$?"
grep -v spmm gpurun_out/landscape.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['schedule'], d['GNZ/s_step'], d['GNZ/s_cached'], d['kernel'][:60])"
