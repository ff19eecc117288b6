# BERT-L P = 4 step (comm_trace's graph-replayed bench step) for DeAR / WFBP
# at larger fusion buffers than the reference's 25 MB default.
mkdir -p gpurun_out
i=0
for buf in 25000000 50000000 100000000; do
  for pol in DEAR_FUSED WFBP_FUSED; do
    i=$((i+1))
    timeout 400 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29800+i)) tools/comm_trace.py --buffer $buf --policy $pol > gpurun_out/r02buf_$i.log 2>&1
    echo "buf=$buf $pol $(grep "^{" gpurun_out/r02buf_$i.log | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['step_ms'],3), d['rs']['launches'])")"
  done
done
