timeout 1500 python -m pytest tests/test_gpu_hot.py -x -q > gpurun_out/pytest_hot.log 2>&1; echo "pytest hot rc=$?"; tail -15 gpurun_out/pytest_hot.log
timeout 900 python tools/sweep_hot.py c3,c5,c4 > gpurun_out/sweep_hot.jsonl 2> gpurun_out/sweep_hot.err; echo "sweep rc=$?"; cat gpurun_out/sweep_hot.jsonl | cut -c1-250; tail -3 gpurun_out/sweep_hot.err
