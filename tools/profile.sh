#!/bin/bash
# Profile recipe (run under gpurun, one GPU). Each ncu pass follows a plain run
# of the same command that exited 0 (B200_PROFILING.md).
#   tools/profile.sh <tag> [bench args...]
set -u
TAG=${1:-r01}
shift || true
OUT=gpurun_out/prof_${TAG}
mkdir -p "$OUT"
CMD=(python bench.py --steps 2 --warmup 1 --no-cpu --no-ablation --profile-steps 2 "$@")
HBM=(python tools/bench_hbm.py --iters 3)
"${CMD[@]}" > "$OUT/plain.log" 2>&1 || { echo "plain run failed"; tail -20 "$OUT/plain.log"; exit 1; }
"${HBM[@]}" > "$OUT/hbm_plain.log" 2>&1 || { echo "hbm plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "dear_profile/" -c 3000 --csv \
    --log-file "$OUT/launches.csv" "${CMD[@]}" > "$OUT/ncu_launches.log" 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "dear_profile/" -k regex:gemm_kernel -s 159 -c 4 \
    -o "$OUT/gemm" "${CMD[@]}" > "$OUT/ncu_gemm.log" 2>&1
ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|update_kernel|unpack_kernel" \
    -s 15 -c 3 -o "$OUT/hbm" "${HBM[@]}" > "$OUT/ncu_hbm.log" 2>&1
echo "profile done: $OUT"
ls -la "$OUT"
