# In-step comm traces (BERT-L, P = 4) for L2-hint / unroll / priority variants.
mkdir -p gpurun_out
i=0
run() {  # lib P [env]
  i=$((i+1))
  env DEAR_LIB=$1 $3 timeout 400 torchrun --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $((29700+i)) tools/comm_trace.py > gpurun_out/r02v3_$i.log 2>&1
  echo "P=$2 $1 $3 $(grep "^{" gpurun_out/r02v3_$i.log | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(round(rows[0][\"step_ms\"],3), \"rs\", [round(r[\"rs\"][\"move_us_median\"],1) for r in rows], \"ag\", [round(r[\"ag\"][\"move_us_median\"],1) for r in rows])")"
}
for rep in 1 2; do
  for lib in libdear.so libdear_ev.so libdear_pu1.so libdear_evpu1.so; do run $lib 4; done
  run libdear.so 4 DEAR_COMM_PRIORITY=low
done
