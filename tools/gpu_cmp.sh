# usage: bash tools/gpu_cmp.sh tag1 tag2 ...   (tag "base" = the in-tree library); two interleaved passes
for pass in 1 2; do for tag in "$@"; do
  if [ $tag = base ]; then lib=paper_2212_08964_b200/liblb.so; else lib=tools/abl/liblb_$tag.so; fi
  LB_LIB_PATH=$lib timeout 300 python bench.py --no-extras --steps 300 --warmup 10 ${BENCH_ARGS} > gpurun_out/cmp.log 2>&1
  echo "pass $pass $tag: $(tail -1 gpurun_out/cmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["phase_ms"]["main"], d.get("no_plan",{}) and d["no_plan"]["value"])' 2>&1 | tail -1)"
done; done
