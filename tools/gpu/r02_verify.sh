# full GPU suite, bench, ncu: warm-L2 C3 capture + per-class DRAM traffic of each class's tile kernel
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r02i_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02i_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; tail -1 gpurun_out/r02i_smoke.log
timeout 900 python bench.py > gpurun_out/r02i_bench.log 2>&1; tail -1 gpurun_out/r02i_bench.log | head -c 1500; echo
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:merge_stream_kernel -s 16 -c 1 \
    -o gpurun_out/r02i_c3_tile_warm python bench.py --steps 3 --warmup 3 --no-extras --classes "" > gpurun_out/r02i_ncu_warm.log 2>&1
for spec in "c2 0 merge_rows" "c2 -1 merge_rows" "c4 0 merge_stream" "c4 -1 merge_stream" "c5 0 merge_stream" "c5 -1 merge_stream" "c3 -1 merge_stream"; do
  set -- $spec
  timeout 600 ncu --metrics $M --clock-control none -k regex:$3 -s 3 -c 1 --csv --log-file gpurun_out/r02i_traffic_$1_$2.csv \
      python tools/prof_run.py $1 $2 5 > gpurun_out/r02i_traffic_$1_$2.log 2>&1
  tail -1 gpurun_out/r02i_traffic_$1_$2.log
done
ls gpurun_out | grep r02i
