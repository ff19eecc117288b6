set -u
mkdir -p gpurun_out
TAG=${1:-r01g}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 > gpurun_out/${TAG}_bench_n4.log 2>&1; echo "bench n4 rc=$?"
grep '"metric"' gpurun_out/${TAG}_bench_n4.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ns=d['north_star']
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['exposed_comm_pct'], d['config']['zero_copy'], d['busbw_gbs'], d['clocks'])
print({k: ns.get(k) for k in ('DEAR_FUSED','WFBP_FUSED','dear_over_wfbp','exposed_comm_pct','compute_only_ms','eq78','buffer_sweep')})
print('cal', {k: (ns.get('calibrated_batch') or {}).get(k) for k in ('batch_per_gpu','dear_over_wfbp','exposed_comm_pct')})
print('nccl', {k: (ns.get('nccl') or {}).get(k) for k in ('dear_over_wfbp','exposed_comm_pct','eq78')})"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --impl reference > gpurun_out/${TAG}_ref_n4.log 2>&1; echo "ref rc=$?"; grep impl gpurun_out/${TAG}_ref_n4.log | cut -c1-400
