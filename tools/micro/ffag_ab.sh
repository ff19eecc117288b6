# Forward-phase all-gathers at unroll 4 (= backprop setting) / 8 / 16, in-step
# (The forward-phase instance, DEAR_PEER_UNROLL_FF, was removed from the product after this measurement.)
# BERT-L traces at P = 4 and P = 2.
mkdir -p gpurun_out
i=0
for rep in 1 2; do
  for lib in libdear_ff4.so libdear.so libdear_ff16.so; do
    for n in 4 2; do
      i=$((i+1))
      dev=0,1,2,3; [ $n = 2 ] && dev=0,1
      CUDA_VISIBLE_DEVICES=$dev DEAR_LIB=$lib timeout 400 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700+i)) tools/comm_trace.py > gpurun_out/r02ffag_$i.log 2>&1
      echo "P=$n $lib $(grep "^{" gpurun_out/r02ffag_$i.log | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(round(rows[0][\"step_ms\"],3), \"ag\", [round(r[\"ag\"][\"move_us_median\"],1) for r in rows])")"
    done
  done
done
