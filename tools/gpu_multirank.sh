# the bench's multi-rank code paths (sharding, all-gather merge, max over ranks, sharded ES) with
# two ranks sharing GPU 0 over gloo (LS_BENCH_SHARED_GPU=1; NCCL refuses two ranks on one device)
for w in conv gemm bert resnet50-es sweep; do
  LS_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --workload $w \
    > gpurun_out/mr_$w.json 2> gpurun_out/mr_$w.err
  echo "$w rc=$?"; tail -n 1 gpurun_out/mr_$w.json | cut -c1-300
done
