# Critical-path collectives (last reduce-scatter, first forward all-gather) on
# the unthrottled instances vs DEAR_CRIT_FAST=0: parity, BERT-L in-step traces
# and the ResNet-50 bench value at P = 4 and 2.
mkdir -p gpurun_out
timeout 600 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29660 tests/dist_worker.py peer > gpurun_out/r02crit_parity_p4.log 2>&1
echo "parity P=4 rc=$? $(grep -c 'bit_exact_fp32_ring=True' gpurun_out/r02crit_parity_p4.log) exact"
CUDA_VISIBLE_DEVICES=0,1 timeout 600 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 tests/dist_worker.py peer > gpurun_out/r02crit_parity_p2.log 2>&1
echo "parity P=2 rc=$? $(grep -c 'bit_exact_fp32_ring=True' gpurun_out/r02crit_parity_p2.log) exact"
i=0
for rep in 1 2; do
  for env in "DEAR_CRIT_FAST=0" "DEAR_CRIT_FAST=1"; do
    for n in 4 2; do
      i=$((i+1)); dev=0,1,2,3; [ $n = 2 ] && dev=0,1
      env CUDA_VISIBLE_DEVICES=$dev $env timeout 400 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+i)) tools/comm_trace.py > gpurun_out/r02crit_tr_$i.log 2>&1
      i=$((i+1))
      env CUDA_VISIBLE_DEVICES=$dev $env timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+i)) bench.py --gpus $n --extra-workload none --buffer-sweep-bytes= --no-parity --no-timeline --no-ablation > gpurun_out/r02crit_b_$i.log 2>&1
      echo "P=$n $env bertl $(grep "^{" gpurun_out/r02crit_tr_$((i-1)).log | head -1 | python -c "import sys,json; print(round(json.loads(sys.stdin.read())['step_ms'],3))") resnet $(grep "^{" gpurun_out/r02crit_b_$i.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],4))")"
    done
  done
done
