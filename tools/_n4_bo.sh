port=29990
for b in peer nccl; do
  port=$((port+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
    tools/tune_fusion_buffer.py --workload bert_base --backend $b --trials 10 > gpurun_out/bo_bert_base_$b.log 2>&1
  grep '^{' gpurun_out/bo_bert_base_$b.log | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('$b', 'best', d['best_buffer_bytes'], round(d['best_samples_per_s']), '25MB', round(d['default_25MB']['samples_per_s']), 'wfbp@best', round(d['wfbp_at_best_buffer']['samples_per_s']), 'wfbp@25', round(d['wfbp_at_25MB']['samples_per_s']), [(t['buffer_bytes']//1000000, round(t['samples_per_s'])) for t in d['trials']])" || tail -5 gpurun_out/bo_bert_base_$b.log
done
