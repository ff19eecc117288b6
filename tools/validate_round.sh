#!/bin/bash
# Round validation on one box (run under `gpurun --gpus 4`): GPU suite (incl.
# the 2- and 4-rank tests), smoke, and the bench at N = 4, 2, 1.
#   tools/validate_round.sh <tag>
set -u
T=${1:-r02z}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${T}_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/${T}_bench_n4.log 2>&1; echo "n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 > gpurun_out/${T}_bench_n2.log 2>&1; echo "n2 rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/${T}_bench_n1.log 2>&1; echo "n1 rc=$?"
timeout 1200 torchrun --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/sweep_collectives.py > gpurun_out/${T}_sweep_p4.log 2>&1; echo "sweep p4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 tools/sweep_collectives.py > gpurun_out/${T}_sweep_p2.log 2>&1; echo "sweep p2 rc=$?"
