#!/bin/bash
# Build diagnostic variants of liblb.so: tools/abl/liblb_<tag>.so for each argument "<tag>:<nvcc -D flags>",
# e.g.  tools/ablate.sh abl1:-DLB_ABL=1 keep:-DLB_HOT_XKEEP=1
# LB_ABL (lb_kernels.cuh) ablations give wrong results by construction (timings only); the other
# switches are candidate changes measured before they are adopted.  Run with LB_LIB_PATH=tools/abl/...
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/abl
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr $flags -I include -o tools/abl/liblb_$tag.so paper_2212_08964_b200/csrc/lb_api.cu -ldl &
done
wait
ls tools/abl
