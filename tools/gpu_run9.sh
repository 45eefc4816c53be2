timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_wide -s 2 -c 1 -o gpurun_out/prof_c2_wide python tools/prof_run.py c2 -1 4 > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 wide rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:thread_mapped -s 2 -c 1 -o gpurun_out/prof_c2_tm python tools/prof_run_sched.py c2 thread_mapped 4 > gpurun_out/ncu_c2tm.log 2>&1; echo "ncu c2 tm rc=$?"
timeout 600 python bench.py --multi --config c3 --steps 20 --warmup 3 --no-extras > gpurun_out/bench_multi1.log 2>&1; echo "multi rc=$?"; tail -1 gpurun_out/bench_multi1.log | cut -c1-1200
