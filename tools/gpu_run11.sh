timeout 1200 python -m pytest tests/test_gpu_fused.py tests/test_gpu_sssp.py -q -x > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_fused.log
