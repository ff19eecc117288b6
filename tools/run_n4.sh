#!/bin/bash
# 4-GPU measurement batch (run under gpurun --gpus 4)
P=${P:-4}
port=29700
for wl in bert_large resnet50; do
  for b in nccl peer; do
    port=$((port+1))
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $P --steps 10 --warmup 3 --no-cpu --workload $wl --backend $b 2>&1 | grep '"metric"'
  done
done
for b in nccl peer; do
  port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
    --master-port $port tools/sweep_collectives.py --backend $b 2>&1 | grep -E '"bytes"|calib'
done
