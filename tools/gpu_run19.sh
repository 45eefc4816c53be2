for tag in base keep; do
  if [ $tag = base ]; then lib=paper_2212_08964_b200/liblb.so; else lib=tools/abl/liblb_$tag.so; fi
  for cc in all none; do
    LB_LIB_PATH=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --cache-control $cc --clock-control none -k regex:merge_stream_kernel -s 20 -c 3 --csv python bench.py --steps 5 --warmup 3 --no-extras 2>/dev/null | grep -E '"(dram|gpu__time|lts)' | awk -F'","' -v t=$tag -v c=$cc '{print t, c, $(NF-2), $NF}'
  done
  LB_LIB_PATH=$lib timeout 300 python bench.py --no-extras --steps 300 --warmup 10 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$tag' bench", d["value"], d["phase_ms"]["main"], d["roofline"]["kernel"])'
done
