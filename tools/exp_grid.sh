#!/bin/bash
# bucket-kernel grid: isolated HBM roofline vs in-step BERT-L (peer backend)
P=${P:-4}
for g in 148 296 592; do
  DEAR_BUCKET_CTAS=$g timeout 120 python tools/bench_hbm.py --workload bert_large --iters 10 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('isolated grid=$g', {k: round(d[k]['frac_of_measured_hbm'],3) for k in ('pack','update','unpack')})"
done
port=29900
for g in 148 296; do
  for b in peer nccl; do
  port=$((port+1))
  DEAR_BUCKET_CTAS=$g timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus $P --steps 10 --warmup 3 \
    --no-cpu --workload bert_large --extra-workload none --backend $b 2>&1 | grep '"metric"' | \
    python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('step grid=$g $b', {'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'compute_ms': round(d['compute_only_ms'],2), 'ratio': round(d['dear_over_wfbp'],3), 'exposed': round(d['exposed_comm_pct'],1), 'wfbp_exposed': round(d['wfbp_exposed_comm_pct'],1)})"
  done
done
