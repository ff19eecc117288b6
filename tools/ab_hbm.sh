#!/bin/bash
# A/B of bucket-kernel variants: event-timed isolation + ncu kernel durations (warm L2).
for lib in "$@"; do
  for w in bert_large resnet50; do
    DEAR_LIB=$lib timeout 120 python tools/bench_hbm.py --workload $w --iters 10 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['workload'], {k: round(d[k]['frac_of_measured_hbm'],3) for k in ('pack','update','unpack')})"
  done
done
for lib in "$@"; do
  DEAR_LIB=$lib timeout 120 python tools/bench_hbm.py --workload bert_large --iters 2 > /dev/null 2>&1 && \
  DEAR_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    -k regex:"pack_kernel|update_kernel|unpack_kernel" --csv --log-file gpurun_out/hbm_${lib}.csv \
    python tools/bench_hbm.py --workload bert_large --iters 2 > /dev/null 2>&1
done
