# GPU-box script: every step under its own timeout (a hang must never eat the call's budget)
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; cat gpurun_out/bench_full.log | tail -1
timeout 300 python tools/sweep_variants.py c3 > gpurun_out/sweep_c3.log 2>&1; cat gpurun_out/sweep_c3.log | tail -9
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"merge|partition|fixup|thread_mapped|group_mapped|validate" --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --no-extras > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:merge_wide -s 3 -c 1 -o gpurun_out/prof_r01_c3 python bench.py --steps 2 --warmup 3 --no-extras > gpurun_out/ncu_run.log 2>&1; echo "ncu full rc=$?"
