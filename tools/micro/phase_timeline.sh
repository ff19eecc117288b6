mkdir -p gpurun_out
for pol in NONE DEAR_FUSED WFBP_FUSED; do
  timeout 400 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29911 tools/graph_timeline.py --workload bert_large --policy $pol --out gpurun_out/r02tl_$pol.json > gpurun_out/r02tl_$pol.log 2>&1
  echo "$pol $(grep '^{' gpurun_out/r02tl_$pol.log | head -1 | cut -c1-600)"
done
