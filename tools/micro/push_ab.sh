# Push reduce-scatter (DEAR_PUSH_RS=1): parity at P = 2 / 4, then in-step
# BERT-L comm traces against the default pull reduce-scatter (P = 4), with the
# push pack's stores per lane per round at 16 (default build) / 4 / 1.
mkdir -p gpurun_out
for n in 2 4; do
  timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29650+n)) tests/dist_worker.py push > gpurun_out/r02push_parity_p$n.log 2>&1
  echo "parity P=$n rc=$? $(grep -c 'bit_exact_fp32_ring=True' gpurun_out/r02push_parity_p$n.log) exact lines; $(grep 'push P' gpurun_out/r02push_parity_p$n.log)"
done
i=0
for rep in 1 2; do
  for cfg in "libdear.so X=0" "libdear.so DEAR_PUSH_RS=1" "libdear_pp4.so DEAR_PUSH_RS=1" "libdear_pp1.so DEAR_PUSH_RS=1"; do
    set -- $cfg
    i=$((i+1))
    env DEAR_LIB=$1 $2 timeout 400 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700+i)) tools/comm_trace.py > gpurun_out/r02push_tr_$i.log 2>&1
    echo "$cfg $(grep "^{" gpurun_out/r02push_tr_$i.log | python -c "
import sys, json
rows=[json.loads(l) for l in sys.stdin]
print(round(rows[0][\"step_ms\"],3), \"rs\", [round(r[\"rs\"][\"move_us_median\"],1) for r in rows], \"ag\", [round(r[\"ag\"][\"move_us_median\"],1) for r in rows])")"
  done
done
