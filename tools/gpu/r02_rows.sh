# short-row kernel + group partition search: parity, A/B timing
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accuracy.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02f_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02f_tests.log
for v in 0 2 4 1 0 2 4 1; do LB_ROWS_VARIANT=$v timeout 300 python tools/ab_rows.py c2; done > gpurun_out/r02f_ab.jsonl 2>&1
cat gpurun_out/r02f_ab.jsonl
