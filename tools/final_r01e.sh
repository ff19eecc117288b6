set -u
TAG=${1:-r01e}
mkdir -p gpurun_out
DEAR_TEST_NPROC=2 timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^\[distoptim|passed|failed" gpurun_out/${TAG}_pytest.log | tail -3
for wl in resnet50 bert_large; do CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/hbm_chain.py --workload $wl 2>&1 | tail -1; done > gpurun_out/${TAG}_hbm_chain.log
cat gpurun_out/${TAG}_hbm_chain.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/${TAG}_bench_n1.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/${TAG}_bench_n1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])
print({k: round(v['frac'],3) for k,v in d['hbm_kernels'].items()})"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/${TAG}_bench_n2.log 2>&1; echo "bench n2 rc=$?"
grep '"metric"' gpurun_out/${TAG}_bench_n2.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); ns=d['north_star']
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['exposed_comm_pct'], d['config']['zero_copy'])
print({k: ns.get(k) for k in ('DEAR_FUSED','WFBP_FUSED','dear_over_wfbp','exposed_comm_pct','compute_only_ms','buffer_sweep')}, (ns.get('calibrated_batch') or {}).get('dear_over_wfbp'), (ns.get('nccl') or {}).get('dear_over_wfbp'))"
