set -u
mkdir -p gpurun_out
N=${N:-2}
tl() {  # tag env... args
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29520 tools/graph_timeline.py $TLARGS > gpurun_out/tl4j_${N}_$tag.log 2>&1; echo "tl $tag rc=$?"
  grep '"rank"' gpurun_out/tl4j_${N}_$tag.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_order'] or {}
print(d['marks_ms'], c.get('stage_us_mean'), d['rs_busy_ms'], d['ag_busy_ms'])"
}
TLARGS="--policy DEAR_FUSED" tl dear X=1
TLARGS="--policy DEAR_FUSED" tl dear_r80 DEAR_LIB=libdear_r80.so
TLARGS="--policy DEAR_FUSED" tl dear_r96 DEAR_LIB=libdear_r96.so
TLARGS="--policy NONE" tl none X=1
