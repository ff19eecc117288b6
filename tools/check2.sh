set -u
mkdir -p gpurun_out
DEAR_TEST_NPROC=2 timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/c2_pytest.log 2>&1; echo "pytest rc=$?"
grep -E "^\[(distoptim|runtime|peer)|passed|failed" gpurun_out/c2_pytest.log | tail -30
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/c2_bench_n1.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/c2_bench_n1.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['frac'])
print(json.dumps(d['hbm_kernels']))"
