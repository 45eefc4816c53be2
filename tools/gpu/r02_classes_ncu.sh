# one ncu --set full capture of each class's default merge-path tile kernel (round-2 final kernels)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_rows -s 3 -c 1 -o gpurun_out/r02cl_c2_rows python tools/prof_run.py c2 0 5 > gpurun_out/r02cl_c2.log 2>&1; tail -1 gpurun_out/r02cl_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 3 -c 1 -o gpurun_out/r02cl_c4_hot python tools/prof_run.py c4 0 5 > gpurun_out/r02cl_c4.log 2>&1; tail -1 gpurun_out/r02cl_c4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:merge_stream -s 3 -c 1 -o gpurun_out/r02cl_c5_hot python tools/prof_run.py c5 0 5 > gpurun_out/r02cl_c5.log 2>&1; tail -1 gpurun_out/r02cl_c5.log
ls gpurun_out | grep r02cl
