set -u
mkdir -p gpurun_out
export DEAR_TEST_NPROC=2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29511 tests/dist_worker.py peer > gpurun_out/zc2_peer.log 2>&1; echo "peer rc=$?"
tail -20 gpurun_out/zc2_peer.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/zc2_bench.log 2>&1; echo "bench rc=$?"
DEAR_ZERO_COPY=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/zc2_bench_slots.log 2>&1; echo "bench slots rc=$?"
for f in gpurun_out/zc2_bench.log gpurun_out/zc2_bench_slots.log; do grep '"metric"' $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ns=d.get('north_star',{})
print(d['value'], d['ms_per_step'], d['config'].get('zero_copy'), d.get('exposed_comm_pct'), d.get('dear_over_wfbp'), d.get('busbw_gbs'))
print('NS', {k: ns.get(k) for k in ('compute_only_ms','DEAR_FUSED','WFBP_FUSED','dear_over_wfbp','exposed_comm_pct','wfbp_exposed_comm_pct','zero_copy')})
print('NCCL', ns.get('nccl'))"; done
