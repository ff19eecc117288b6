# P = 2 reduce-scatter vectors per lane per round: 1 (default) vs 2, in-step
# BERT-L traces and the ResNet-50 bench value.
mkdir -p gpurun_out
i=0
for rep in 1 2 3; do
  for lib in libdear.so libdear_ku22.so; do
    i=$((i+1))
    DEAR_LIB=$lib timeout 400 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29700+i)) tools/comm_trace.py > gpurun_out/r02ku2_tr_$i.log 2>&1
    DEAR_LIB=$lib timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29750+i)) bench.py --gpus 2 --extra-workload none --buffer-sweep-bytes= --no-parity --no-timeline --no-ablation > gpurun_out/r02ku2_b_$i.log 2>&1
    echo "$lib bertl $(grep "^{" gpurun_out/r02ku2_tr_$i.log | head -1 | python -c "import sys,json; print(round(json.loads(sys.stdin.read())['step_ms'],3))") resnet $(grep "^{" gpurun_out/r02ku2_b_$i.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']))")"
  done
done
