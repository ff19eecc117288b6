set -u
mkdir -p gpurun_out
N=${N:-4}
export DEAR_TEST_NPROC=$N
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29511 tests/dist_worker.py peer > gpurun_out/zc4_peer.log 2>&1; echo "peer rc=$?"
grep "^\[peer" gpurun_out/zc4_peer.log
tl() {  # tag env... args
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port 29520 tools/graph_timeline.py $TLARGS > gpurun_out/tl4_$tag.log 2>&1; echo "tl $tag rc=$?"
  grep '"rank"' gpurun_out/tl4_$tag.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_order'] or {}
print(d['marks_ms'], c.get('ags_during_backprop'), c.get('stage_us_mean'), d['rs_busy_ms'], d['ag_busy_ms'])"
}
TLARGS="--policy NONE" tl none X=1
TLARGS="--policy DEAR_FUSED --group-dependency 0" tl dear_gd0 X=1
TLARGS="--policy NONE" tl none_cap132 DEAR_GEMM_MAX_CTAS=132
TLARGS="--policy DEAR_FUSED" tl dear_part DEAR_GEMM_MAX_CTAS=132 DEAR_LIB=libdear_part.so
TLARGS="--policy NONE" tl none_cap140 DEAR_GEMM_MAX_CTAS=140
TLARGS="--policy DEAR_FUSED" tl dear_part140 DEAR_GEMM_MAX_CTAS=140 DEAR_LIB=libdear_part.so
