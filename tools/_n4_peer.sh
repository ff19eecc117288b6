timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/sweep_collectives.py --backend peer 2>&1 | grep '^{' | python3 -c "
import sys,json
for l in sys.stdin:
  d=json.loads(l)
  if d['bytes'] in (4194304, 16777216, 33554432, 268435456): print({k:(round(v,1) if isinstance(v,float) else v) for k,v in d.items()})"
SKIP_TESTS=1 CTS=1.0 bash tools/n4_gd.sh
