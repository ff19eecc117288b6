set -u
mkdir -p gpurun_out
for buf in 5000000 10000000 25000000 50000000; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --buffer $buf --no-cpu --extra-workload none > gpurun_out/bs4_$buf.log 2>&1; echo "buf $buf rc=$?"
grep '"metric"' gpurun_out/bs4_$buf.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['exposed_comm_pct'], d['config']['buckets'], d.get('dear_over_wfbp'), d['compute_only_ms'])"
done
