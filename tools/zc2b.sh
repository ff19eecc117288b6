set -u
mkdir -p gpurun_out
export DEAR_TEST_NPROC=2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29511 tests/dist_worker.py peer > gpurun_out/zc2b_peer.log 2>&1; echo "peer rc=$?"
grep "^\[peer" gpurun_out/zc2b_peer.log
for pol in NONE DEAR_FUSED WFBP_FUSED; do
for gd in 1; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29520 tools/graph_timeline.py --policy $pol --group-dependency $gd --out gpurun_out/tl2_${pol}.json > gpurun_out/tl2_${pol}.log 2>&1; echo "tl $pol rc=$?"
grep '"rank"' gpurun_out/tl2_${pol}.log | cut -c1-900
done; done
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/zc2b_bench.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/zc2b_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ns=d.get('north_star',{})
print(d['value'], d['ms_per_step'], d['config'].get('zero_copy'), d.get('exposed_comm_pct'), d.get('dear_over_wfbp'), d.get('busbw_gbs'))
print(json.dumps(d.get('hbm_kernels')))
print(json.dumps(ns))"
