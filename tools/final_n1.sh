#!/bin/bash
# One-GPU round-end evidence: GPU tests, smoke, default bench, then the ncu pass
# (tools/profile.sh: launch list + GEMM/HBM full captures).
set -u
TAG=${1:-r01c}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/${TAG}_bench.log | cut -c1-600
bash tools/profile.sh "$TAG" --extra-workload none
