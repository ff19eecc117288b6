port=29800
for pol in DEAR_FUSED WFBP_FUSED; do
port=$((port+1))
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $port \
  tools/trace_step.py --workload bert_large --policy $pol --backend peer --out gpurun_out/trace 2>&1 | grep -v Warning | tail -3
done
