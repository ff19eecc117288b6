port=29870
run() { # tag env... -- args
  tag=$1; shift
  port=$((port+1))
  env "$@" timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --workload bert_large \
    --extra-workload none $BARGS > gpurun_out/n4_v2_$tag.log 2>&1
  grep '"metric"' gpurun_out/n4_v2_$tag.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); o=d['config']['comm_order'] or {}; print('$tag', {'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'compute_ms': round(d['compute_only_ms'],2), 'ratio': round(d['dear_over_wfbp'],3), 'exposed': round(d['exposed_comm_pct'],1), 'ags_bp': o.get('ags_during_backprop'), 'stage_us': {k: round(v,1) for k,v in (o.get('stage_us_mean') or {}).items()}})"
}
run grid148_ct1.0 X=1
BARGS="--contention 0.7" run grid148_ct0.7 X=1
run grid592_ct1.0 DEAR_BUCKET_CTAS=592
BARGS="--contention 0.7" run grid592_ct0.7 DEAR_BUCKET_CTAS=592
