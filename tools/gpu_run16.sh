timeout 600 ncu --set full --clock-control none --import-source on -k regex:probe_stream -s 1 -c 1 -o gpurun_out/prof_c3_probe_hot python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu16a.log 2>&1; echo "ncu probe rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:merge_stream_kernel -s 20 -c 1 -o gpurun_out/prof_c3_hot python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/ncu16b.log 2>&1; echo "ncu main rc=$?"
ls -la gpurun_out/*.ncu-rep
