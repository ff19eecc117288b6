port=29910
for b in nccl peer; do
  port=$((port+1))
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --workload bert_large \
    --extra-workload none --backend $b --order-search 0 > gpurun_out/n4_stage_$b.log 2>&1
  grep '"metric"' gpurun_out/n4_stage_$b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); o=d['config']['comm_order'] or {}; print('$b', {'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'ratio': round(d['dear_over_wfbp'],3), 'stage_us': {k: round(v,1) for k,v in o.get('stage_us_mean',{}).items()}, 'hbm': {k: round(v['ms_per_step']*1e3/57,1) for k,v in d['hbm_kernels'].items()}})"
done
