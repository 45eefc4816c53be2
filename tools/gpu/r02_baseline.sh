# round-2 baseline on the restored tree: GPU tests, smoke, bench, reference arm, launch list, full ncu of the tile kernel
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r02a_gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r02a_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1; tail -2 gpurun_out/r02a_smoke.log
timeout 600 python bench.py > gpurun_out/r02a_bench.log 2>&1; tail -1 gpurun_out/r02a_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/r02a_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_stream_kernel -s 16 -c 1 \
    -o gpurun_out/r02a_tile_full python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/r02a_full.log 2>&1
ls -la gpurun_out
