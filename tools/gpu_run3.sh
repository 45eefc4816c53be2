export LB_HOT_W=16
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 2 -c 1 -o gpurun_out/prof_c3_hot16k python tools/prof_run.py c3 16384 4 > gpurun_out/ncu_hot.log 2>&1; echo "ncu hot rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 2 -c 1 -o gpurun_out/prof_c3_hot32k python tools/prof_run.py c3 32768 4 > gpurun_out/ncu_hot32.log 2>&1; echo "ncu hot32 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 2 -c 1 -o gpurun_out/prof_c3_base python tools/prof_run.py c3 -1 4 > gpurun_out/ncu_base.log 2>&1; echo "ncu base rc=$?"
