timeout 1200 python -m pytest tests/test_gpu_sssp.py -q > gpurun_out/pytest_sssp.log 2>&1; echo "pytest sssp rc=$?"; tail -15 gpurun_out/pytest_sssp.log
true
