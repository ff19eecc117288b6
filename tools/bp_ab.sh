set -u
mkdir -p gpurun_out
for sp in 0 1; do
for wl in resnet50 bert_large; do
DEAR_BP_SPLIT=$sp timeout 600 python bench.py --no-cpu --no-ablation --extra-workload none --workload $wl --steps 10 > gpurun_out/bpab_${sp}_$wl.log 2>&1; echo "split=$sp $wl rc=$?"
grep '"metric"' gpurun_out/bpab_${sp}_$wl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), round(d['compute_only_ms'],3), round(d['roofline']['frac'],3), json.dumps(d['gemm_tiles']))"
done; done
