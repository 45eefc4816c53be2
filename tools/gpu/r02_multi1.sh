# the multi-GPU bench path at world size 1 (torchrun, NCCL): plain, chunked overlap, fused epilogue
for extra in "" "--overlap" "--fused"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus 1 --multi --config c5 --steps 20 --warmup 3 $extra > gpurun_out/r02v_multi1$extra.log 2>&1; echo "rc=$? $extra"
  tail -1 gpurun_out/r02v_multi1$extra.log | head -c 700; echo
done
