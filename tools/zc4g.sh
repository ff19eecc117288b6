set -u
mkdir -p gpurun_out
N=${N:-4}
tl() {  # tag env... args
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29520 tools/graph_timeline.py $TLARGS > gpurun_out/tl4g_$tag.log 2>&1; echo "tl $tag rc=$?"
  grep '"rank"' gpurun_out/tl4g_$tag.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_order'] or {}
print(d['marks_ms'], c.get('ags_during_backprop'), c.get('stage_us_mean'), c.get('buckets'), d['rs_busy_ms'], d['ag_busy_ms'])"
}
for buf in 50000000 100000000 200000000; do
TLARGS="--policy DEAR_FUSED --buffer $buf" tl dear_$buf X=1
TLARGS="--policy WFBP_FUSED --buffer $buf" tl wfbp_$buf X=1
done
