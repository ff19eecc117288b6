port=29890
for i in 1 2; do
  port=$((port+1))
  timeout 500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $port bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu --workload bert_large \
    --extra-workload none > gpurun_out/n4_search_$i.log 2>&1
  grep '"metric"' gpurun_out/n4_search_$i.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); o=d['config']['comm_order'] or {}; print('run$i', {'dear_ms': round(d['ms_per_step'],2), 'wfbp_ms': round(d['wfbp']['ms_per_step'],2), 'compute_ms': round(d['compute_only_ms'],2), 'ratio': round(d['dear_over_wfbp'],3), 'exposed': round(d['exposed_comm_pct'],1), 'chosen': o.get('ags_during_backprop'), 'cands': [(c['ags_during_backprop'], round(c['ms'],2), round(c['predicted_ms'],2)) for c in o.get('candidates', [])]})"
done
