timeout 120 python tools/pcie_probe.py > gpurun_out/r02l_pcie.json 2>&1; cat gpurun_out/r02l_pcie.json
timeout 1500 python tools/bench_matrix.py c1,c2,c3,c4,c5 > gpurun_out/r02l_landscape.jsonl 2>&1; tail -3 gpurun_out/r02l_landscape.jsonl
