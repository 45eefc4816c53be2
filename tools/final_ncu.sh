# final-tree evidence: launch list of the bench command + one full capture of the C3 tile kernel
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/f_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:merge_stream_kernel -s 16 -c 1 \
    -o gpurun_out/f_tile_full python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/f_full.log 2>&1
ls -la gpurun_out
