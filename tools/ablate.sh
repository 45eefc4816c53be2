#!/bin/bash
# Build diagnostic ablation libraries of liblb.so (tools/abl/liblb_<mask>.so, see LB_ABL in
# lb_kernels.cuh) -- timings only, the results are wrong by construction.
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/abl
for m in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr -DLB_ABL=$m -I include -o tools/abl/liblb_$m.so paper_2212_08964_b200/csrc/lb_api.cu -ldl &
done
wait
ls tools/abl
