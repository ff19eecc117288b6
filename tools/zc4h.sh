set -u
mkdir -p gpurun_out
N=${N:-4}
tl() {  # tag env... args
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29520 tools/graph_timeline.py $TLARGS > gpurun_out/tl4h_$tag.log 2>&1; echo "tl $tag rc=$?"
  grep '"rank"' gpurun_out/tl4h_$tag.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_order'] or {}
print(d['marks_ms'], d['clocks'], d['rs_busy_ms'], d['ag_busy_ms'])"
}
TLARGS="--policy NONE --clock-steps 400" tl none X=1
TLARGS="--policy DEAR_FUSED --clock-steps 400" tl dear X=1
