timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep_hot.py c3,c4,c5,c2 8192,16384,24576,32768 8,16 1016 > gpurun_out/sweep_hot2.jsonl 2> gpurun_out/sweep_hot2.err; echo "sweep rc=$?"; cut -c1-250 gpurun_out/sweep_hot2.jsonl; tail -3 gpurun_out/sweep_hot2.err
