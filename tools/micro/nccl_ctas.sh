# NCCL CTA caps vs the BERT-L DeAR / WFBP step on the NCCL transport (N = 4);
# the first run is the full default bench line (incl. the config-3 sweep).
mkdir -p gpurun_out
i=0
for env in "X=0" "NCCL_MAX_CTAS=16" "NCCL_MAX_CTAS=8" "NCCL_MAX_CTAS=4" "NCCL_MAX_CTAS=2"; do
  i=$((i+1))
  extra=""; [ $i -gt 1 ] && extra="--buffer-sweep-bytes= --no-priority-partition --no-parity --no-timeline"
  env $env timeout 900 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus 4 $extra > gpurun_out/r02nc_$i.log 2>&1
  echo "$env $(grep '^{' gpurun_out/r02nc_$i.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); n=d['north_star']['nccl']
print('dear', round(n['DEAR_FUSED']['ms_per_step'],3), 'wfbp', round(n['WFBP_FUSED']['ms_per_step'],3), 't_rs', round(n['t_rs_ms'],3), 't_ag', round(n['t_ag_ms'],3), 'peer', round(d['north_star']['DEAR_FUSED']['ms_per_step'],3))")"
done
