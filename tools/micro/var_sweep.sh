mkdir -p gpurun_out
i=0
run() {  # lib P
  i=$((i+1))
  DEAR_LIB=$1 timeout 400 torchrun --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $((29700+i)) tools/comm_trace.py > gpurun_out/r02v2_$i.log 2>&1
  echo "P=$2 $1 $(grep "^{" gpurun_out/r02v2_$i.log | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(round(rows[0][\"step_ms\"],3), \"rs\", [round(r[\"rs\"][\"move_us_median\"],1) for r in rows], \"ag\", [round(r[\"ag\"][\"move_us_median\"],1) for r in rows])")"
}
for rep in 1 2; do
  for lib in libdear.so libdear_ku1.so libdear_pu4.so libdear_ku1pu4.so libdear_ku1pu2.so; do run $lib 4; done
done
for rep in 1 2; do
  for lib in libdear.so libdear_ku1pu4.so libdear_ku1pu4k2.so libdear_ku1pu4k21.so; do CUDA_VISIBLE_DEVICES=0,1 run $lib 2; done
done
