for v in 1; do LB_SHORT_KERNEL=$v timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accuracy.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02o_tests_v$v.log 2>&1; echo "tests v$v rc=$?"; tail -4 gpurun_out/r02o_tests_v$v.log; done
for v in 0 1 2 3 0 1 2 3; do LB_SHORT_KERNEL=$v timeout 300 python tools/ab_rows.py c2,c4; done > gpurun_out/r02o_ab.jsonl 2>&1
cat gpurun_out/r02o_ab.jsonl
