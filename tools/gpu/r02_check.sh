timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r02x_gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02x_gpu_tests.log
