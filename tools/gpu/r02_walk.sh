LB_SHORT_KERNEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accuracy.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02h_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r02h_tests.log
for v in 0 1 2 0 1 2; do LB_SHORT_KERNEL=$v timeout 300 python tools/ab_rows.py c2,c4; done > gpurun_out/r02h_ab.jsonl 2>&1
cat gpurun_out/r02h_ab.jsonl
