#!/bin/bash
# Compute/comm interference matrix on BERT-L at P GPUs (run under gpurun --gpus P).
P=${P:-4}
port=29800
run() {
  port=$((port+1))
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P \
    --master-addr 127.0.0.1 --master-port $port bench.py --gpus $P --steps 10 --warmup 3 \
    --no-cpu --workload bert_large --extra-workload none ${BENCH_ARGS:-} 2>&1 | grep '"metric"' | \
    python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('$*', {'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'compute_ms': round(d['compute_only_ms'],2), 'ratio': round(d['dear_over_wfbp'],3), 'exposed': round(d['exposed_comm_pct'],1), 'busbw': d.get('busbw_gbs')})"
}
run X=baseline
run DEAR_GEMM_MAX_CTAS=132
run DEAR_BUCKET_CTAS=148
run DEAR_BUCKET_CTAS=148 DEAR_GEMM_MAX_CTAS=140
run NCCL_MAX_CTAS=8
run NCCL_MAX_CTAS=8 DEAR_BUCKET_CTAS=148
BENCH_ARGS="--backend peer" run DEAR_BUCKET_CTAS=148
