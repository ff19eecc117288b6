bash tools/validate_round.sh r02w
for i in 1 2; do
  CUDA_VISIBLE_DEVICES=0,1 timeout 900 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29530+i)) bench.py --gpus 2 > gpurun_out/r02w_bench_n2_rep$i.log 2>&1; echo "n2 rep$i rc=$? $(grep -c '^{' gpurun_out/r02w_bench_n2_rep$i.log) lines $(grep -o '"error": "[^"]*' gpurun_out/r02w_bench_n2_rep$i.log | head -2)"
done
