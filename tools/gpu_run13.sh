for m in 0 1 2 4 7; do
  if [ $m = 0 ]; then lib=paper_2212_08964_b200/liblb.so; else lib=tools/abl/liblb_$m.so; fi
  LB_LIB_PATH=$lib timeout 300 python bench.py --no-extras --steps 100 --warmup 5 > gpurun_out/abl_$m.log 2>&1
  echo "abl $m: $(tail -1 gpurun_out/abl_$m.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["no_plan"]["value"], d["phase_ms"], d["roofline"]["kernel"])')"
done
