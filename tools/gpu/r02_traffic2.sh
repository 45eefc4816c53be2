M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for cfg in c3 c4 c5; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:merge_stream -s 3 -c 1 --csv --log-file gpurun_out/r02y_traffic_${cfg}_-1.csv \
      python tools/prof_run.py $cfg -1 5 > gpurun_out/r02y_traffic_${cfg}.log 2>&1; tail -1 gpurun_out/r02y_traffic_${cfg}.log
done
timeout 900 python bench.py > gpurun_out/r02y_bench.log 2>&1; tail -1 gpurun_out/r02y_bench.log | head -c 300
