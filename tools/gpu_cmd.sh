# GPU-box script: every step under its own timeout (a hang must never eat the call's budget)
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for L in 1016 2040 3064 4088; do timeout 180 python bench.py --steps 200 --warmup 5 --no-extras --items-per-tile $L > gpurun_out/bench_L$L.log 2>&1; done
for c in c2 c4; do timeout 180 python bench.py --steps 100 --warmup 5 --no-extras --config $c > gpurun_out/bench_$c.log 2>&1; done
for f in gpurun_out/bench_*.log; do echo $f; cut -c1-120 $f; grep -o '"phase_ms.*' $f | cut -c1-150; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:merge_pipe -s 3 -c 1 -o gpurun_out/prof_pipe_r01c python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_run.log 2>&1; echo "ncu rc=$?"
