#!/bin/bash
# 4-GPU check: BERT-L (north-star config) DeAR vs WFBP, peer and NCCL backends;
# default bench (ResNet-50) at N=4.
P=${P:-4}
port=29700
for b in peer nccl; do
  port=$((port+1))
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus $P --steps 10 --warmup 3 --no-cpu --workload bert_large \
    --extra-workload none --backend $b > gpurun_out/n4_bertl_$b.log 2>&1
  grep '"metric"' gpurun_out/n4_bertl_$b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('bert_large $b', {'value': round(d['value']), 'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'compute_ms': round(d['compute_only_ms'],2), 'ratio': round(d['dear_over_wfbp'],3), 'exposed': round(d['exposed_comm_pct'],1), 'wfbp_exposed': round(d['wfbp_exposed_comm_pct'],1), 'clocks': d['clocks']})"
done
port=$((port+1))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
  --master-port $port bench.py --gpus $P > gpurun_out/n4_default.log 2>&1
grep '"metric"' gpurun_out/n4_default.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('default', {'value': round(d['value']), 'ms': round(d['ms_per_step'],2), 'ratio': round(d.get('dear_over_wfbp',0),3), 'exposed': round(d['exposed_comm_pct'],1), 'ns': d.get('north_star')})"
