#!/bin/bash
# ncu durations of the bucket kernels (pack/update/unpack), cold and warm L2.
#   tools/profile_hbm.sh <tag> [workload]
set -u
TAG=${1:-r01}; WL=${2:-bert_large}
OUT=gpurun_out/prof_${TAG}; mkdir -p "$OUT"
CMD=(python tools/bench_hbm.py --workload "$WL" --iters 2)
"${CMD[@]}" > "$OUT/hbm_plain_${WL}.log" 2>&1 || { echo "plain failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"pack_kernel|update_kernel|unpack_kernel" --csv --log-file "$OUT/hbm_cold_${WL}.csv" "${CMD[@]}" > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
    -k regex:"pack_kernel|update_kernel|unpack_kernel" --csv --log-file "$OUT/hbm_warm_${WL}.csv" "${CMD[@]}" > /dev/null 2>&1
echo done; ls -la "$OUT"
