LB_SHORT_KERNEL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02p_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02p_tests.log
for v in 0 1 0 1 0 1; do LB_SHORT_KERNEL=$v timeout 300 python tools/ab_rows.py c2; done > gpurun_out/r02p_ab.jsonl 2>&1
cat gpurun_out/r02p_ab.jsonl | cut -c1-200
