set -u
mkdir -p gpurun_out
for be in peer nccl; do
for buf in 5000000 10000000 25000000; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --workload bert_base --buffer $buf --backend $be --no-cpu --extra-workload none --steps 10 > gpurun_out/bb4_${be}_$buf.log 2>&1; echo "$be buf $buf rc=$?"
grep '"metric"' gpurun_out/bb4_${be}_$buf.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), 'wfbp', round(d['wfbp']['ms_per_step'],3), 'dear/wfbp', round(d.get('dear_over_wfbp'),3), 'exposed', round(d['exposed_comm_pct'],1), round(d['wfbp_exposed_comm_pct'],1), 'buckets', d['config']['buckets'], 'compute', round(d['compute_only_ms'],3))"
done; done
