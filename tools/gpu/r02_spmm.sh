timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_accuracy.py -m gpu -q -x -p no:cacheprovider -k "spmm" > gpurun_out/r02s_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02s_tests.log
for lib in "" tools/abl/liblb_blk1.so "" tools/abl/liblb_blk1.so; do echo "lib=${lib:-default}"; LB_LIB_PATH=$lib timeout 600 python tools/bench_spmm.py c3,c4 4,8 ; done > gpurun_out/r02s_spmm.txt 2>&1
cat gpurun_out/r02s_spmm.txt
