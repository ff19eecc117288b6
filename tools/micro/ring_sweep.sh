# GEMM ring 102 KB vs 96 KB: with 102 KB two GEMM CTAs fill an SM's shared
# memory and a comm CTA (1 KB static + 1 KB reserved) cannot co-reside.
mkdir -p gpurun_out
i=0
run() {  # lib P [env]
  i=$((i+1))
  env DEAR_LIB=$1 $3 timeout 400 torchrun --nproc-per-node $2 --master-addr 127.0.0.1 --master-port $((29800+i)) tools/comm_trace.py > gpurun_out/r02v4_$i.log 2>&1
  echo "P=$2 $1 $3 $(grep "^{" gpurun_out/r02v4_$i.log | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(round(rows[0][\"step_ms\"],3), \"rs\", [round(r[\"rs\"][\"move_us_median\"],1) for r in rows], \"ag\", [round(r[\"ag\"][\"move_us_median\"],1) for r in rows])")"
}
for rep in 1 2; do
  for lib in libdear.so libdear_r96.so; do run $lib 4; done
done
for lib in libdear.so libdear_r96.so; do
  DEAR_LIB=$lib timeout 600 python bench.py --no-parity --no-timeline > gpurun_out/r02v4_n1_$lib.log 2>&1
  echo "N=1 $lib $(grep '^{' gpurun_out/r02v4_n1_$lib.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['gemm_tiles'])")"
done
