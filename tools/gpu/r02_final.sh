# final-tree verification: GPU suite, smoke, bench (+ reference arm), launch list + one full ncu capture
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r02z_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02z_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.log 2>&1; tail -1 gpurun_out/r02z_smoke.log
timeout 900 python bench.py > gpurun_out/r02z_bench.log 2>&1; tail -1 gpurun_out/r02z_bench.log | head -c 400; echo
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02z_bench_ref.log 2>&1; tail -1 gpurun_out/r02z_bench_ref.log | head -c 300; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02z_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-extras --classes "" > gpurun_out/r02z_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_stream_kernel -s 16 -c 1 \
    -o gpurun_out/r02z_tile_full python bench.py --steps 3 --warmup 3 --no-extras --classes "" > gpurun_out/r02z_full.log 2>&1
ls gpurun_out | grep r02z
