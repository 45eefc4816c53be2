timeout 1200 python -m pytest tests/test_gpu_multi_procs.py -m gpu -q -p no:cacheprovider > gpurun_out/r02q_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/r02q_tests.log
