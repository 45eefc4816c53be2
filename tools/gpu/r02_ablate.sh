# ablations of the C3 hot tile kernel (results wrong by construction, timings only): graph-replayed step
for lib in "" tools/abl/liblb_abl1.so tools/abl/liblb_abl2.so tools/abl/liblb_abl4.so tools/abl/liblb_abl7.so "" ; do
  LB_LIB_PATH=$lib timeout 300 python bench.py --steps 200 --warmup 10 --no-extras --classes "" | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lib=${lib:-full}', d['value'], d['graph']['value'], round(d['phase_ms']['main'],4))"
done 2>&1 | tee gpurun_out/r02ag_ablate.txt
