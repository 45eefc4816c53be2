timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "graph" > gpurun_out/pt21.log 2>&1; echo "graph tests rc=$?"; tail -3 gpurun_out/pt21.log
timeout 900 python tools/bench_matrix.py c1,c2,c3,c4,c5 > gpurun_out/landscape.jsonl 2> gpurun_out/landscape.err; echo "landscape rc=$?"; tail -3 gpurun_out/landscape.err
grep -v spmm gpurun_out/landscape.jsonl | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['schedule'], d['GNZ/s_step'], d['GNZ/s_cached'], d['GNZ/s_graph'], d['ms_graph'], d['kernel'][:40])"
