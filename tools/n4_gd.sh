#!/bin/bash
# 4 GPUs: parity (runtime + multi-GPU incl. group dependency), then BERT-L DeAR
# with dear_group_dependency (simulated dispatch order, several contention
# factors) vs the global-barrier DeAR vs WFBP, peer backend.
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 900 python -m pytest tests/test_runtime_gpu.py tests/test_multigpu.py -x -q 2>&1 | tail -3
fi
port=29750
run() {  # gd ct
  port=$((port+1))
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --workload ${WL:-bert_large} \
    --extra-workload none --group-dependency $1 --contention $2 > gpurun_out/n4_gd$1_ct$2.log 2>&1
  grep '"metric"' gpurun_out/n4_gd$1_ct$2.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('gd=$1 ct=$2', {'value': round(d['value']), 'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'compute_ms': round(d['compute_only_ms'],2), 'ratio': round(d['dear_over_wfbp'],3), 'exposed': round(d['exposed_comm_pct'],1), 'order': d['config'].get('comm_order')})"
}
for ct in ${CTS:-1.0 1.3 1.6}; do run 1 $ct; done
run 0 1.0
