#!/bin/bash
# Build diagnostic variants of liblb.so: tools/abl/liblb_<tag>.so for each argument "<tag>:<nvcc -D flags>",
# e.g.  tools/ablate.sh abl1:-DLB_ABL=1
# LB_ABL (dev_common.cuh) ablations give wrong results by construction (timings only); other switches
# are candidate changes measured before they are adopted.  Run with LB_LIB_PATH=tools/abl/...
set -e
cd "$(dirname "$0")/.."
mkdir -p tools/abl
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  python -c "
import sys; sys.path.insert(0, '.')
from paper_2212_08964_b200 import build
build.OBJDIR = 'tools/abl/obj_$tag'
build.build(force=True, out='tools/abl/liblb_$tag.so', extra='$flags'.split())"
done
ls tools/abl
