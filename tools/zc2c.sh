set -u
mkdir -p gpurun_out
for lib in ${LIBS:-libdear_ps148k8.so libdear_skipag.so libdear_skipall.so}; do
DEAR_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29520 tools/graph_timeline.py --policy DEAR_FUSED --group-dependency 1 > gpurun_out/tl2c_$lib.log 2>&1; echo "tl $lib rc=$?"
grep '"rank"' gpurun_out/tl2c_$lib.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['comm_order'] or {}
print(d['marks_ms'], c.get('ags_during_backprop'), c.get('stage_us_mean'), d['rs_busy_ms'], d['ag_busy_ms'])"
done
