timeout 900 python -m pytest tests/test_gpu_hot.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02g_tests.log
timeout 600 python tools/probe_cluster.py c3 > gpurun_out/r02g_probe_cluster.jsonl 2>&1; cat gpurun_out/r02g_probe_cluster.jsonl
timeout 900 python bench.py > gpurun_out/r02g_bench.log 2>&1; tail -1 gpurun_out/r02g_bench.log | head -c 6000
