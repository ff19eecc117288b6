port=29770
for cfg in "DEAR_FUSED 1" "DEAR_FUSED 0" "WFBP_FUSED 0"; do
  set -- $cfg; port=$((port+1))
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
    tools/graph_timeline.py --policy $1 --group-dependency $2 --out gpurun_out/tl_$1_$2.json > gpurun_out/tl_$1_$2.log 2>&1
  grep '^{' gpurun_out/tl_$1_$2.log | cut -c1-900 || grep -A3 Traceback gpurun_out/tl_$1_$2.log | head -20
done
