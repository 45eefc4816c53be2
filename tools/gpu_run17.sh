for pdl in 1 0; do
  LB_PDL=$pdl timeout 300 python bench.py --no-extras --steps 300 --warmup 10 > gpurun_out/pdl.log 2>&1
  echo "PDL $pdl: $(tail -1 gpurun_out/pdl.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["phase_ms"], d["no_plan"])')"
done
timeout 300 nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
