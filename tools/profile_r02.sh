#!/bin/bash
# Round-2 profile recipe (one GPU, under gpurun). Each ncu pass follows a plain
# run of the same command that exited 0 (B200_PROFILING.md).
#   tools/profile_r02.sh <tag>
set -u
TAG=${1:-r02}
OUT=gpurun_out/prof_${TAG}
mkdir -p "$OUT"
CMD=(python bench.py --steps 2 --warmup 1 --no-cpu --no-ablation --no-parity --no-timeline
     --extra-workload none --profile-steps 2)
TC=gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__inst_executed_pipe_tc.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts_mem_shared_op_utcmma_matrix_a.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
"${CMD[@]}" > "$OUT/plain.log" 2>&1 || { echo "plain run failed"; tail -20 "$OUT/plain.log"; exit 1; }
# 1. launch list of two graph-replayed steps (serialised, cold caches)
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "dear_profile/" \
    -c 3000 --csv --log-file "$OUT/launches.csv" "${CMD[@]}" > "$OUT/ncu_launches.log" 2>&1
# 2. the whole step as ONE graph workload: in-graph (overlapped) tensor-pipe and
#    TMEM activity, L2 / DRAM bytes — reconciles per-launch ncu times with the graph
ncu --graph-profiling graph --metrics "$TC" --clock-control none --nvtx --nvtx-include "dear_profile/" \
    -c 2 --csv --log-file "$OUT/graph_tc.csv" "${CMD[@]}" > "$OUT/ncu_graph.log" 2>&1
# 3. per-launch tcgen05 metrics of the first FF and BP GEMMs of a step
ncu --metrics "$TC" --clock-control none --nvtx --nvtx-include "dear_profile/" -k regex:gemm_kernel \
    -c 8 --csv --log-file "$OUT/gemm_tc.csv" "${CMD[@]}" > "$OUT/ncu_gemm_tc.log" 2>&1
# 4. full set on one FF and one BP launch
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "dear_profile/" \
    -k regex:gemm_kernel -s 160 -c 2 -o "$OUT/gemm" "${CMD[@]}" > "$OUT/ncu_gemm.log" 2>&1
ncu -i "$OUT/gemm.ncu-rep" --page raw --csv > "$OUT/gemm_full_raw.csv" 2>/dev/null
# 5. bucket kernels (PDL chain tool), full set
HBM=(python tools/hbm_chain.py --reps 3)
"${HBM[@]}" > "$OUT/hbm_plain.log" 2>&1
ncu --set full --clock-control none -k regex:"pack_kernel|update_kernel|unpack_kernel|update_direct" \
    -s 20 -c 4 -o "$OUT/hbm" "${HBM[@]}" > "$OUT/ncu_hbm.log" 2>&1
ncu -i "$OUT/hbm.ncu-rep" --page raw --csv > "$OUT/hbm_full_raw.csv" 2>/dev/null
echo "profile done: $OUT"
ls -la "$OUT"
