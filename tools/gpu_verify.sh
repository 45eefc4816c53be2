# full verification of the tree on one B200: gpu tests, smoke, default bench line
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/v_pt.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/v_pt.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/v_smoke.log
timeout 600 python bench.py > gpurun_out/v_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/v_bench.log
timeout 300 python bench.py --impl reference > gpurun_out/v_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/v_ref.log
