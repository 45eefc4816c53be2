timeout 600 ./tools/mb_cpasync > gpurun_out/mb_cpasync.txt 2>&1; echo "mb rc=$?"; cat gpurun_out/mb_cpasync.txt
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-extras > gpurun_out/bench_c5.log 2>&1; echo "bench c5 rc=$?"; tail -1 gpurun_out/bench_c5.log | cut -c1-1500
