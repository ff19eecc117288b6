set -u
mkdir -p gpurun_out
for lib in ${LIBS:-libdear.so libdear_g2.so}; do
DEAR_LIB=$lib timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q > gpurun_out/gab_$lib.log 2>&1; echo "$lib gemm tests rc=$?"; tail -1 gpurun_out/gab_$lib.log
DEAR_LIB=$lib timeout 600 python bench.py --no-cpu --no-ablation --extra-workload none > gpurun_out/gab_bench_$lib.log 2>&1; echo "bench rc=$?"
grep '"metric"' gpurun_out/gab_bench_$lib.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], json.dumps(d['gemm_tiles']))"
DEAR_LIB=$lib timeout 600 python bench.py --no-cpu --no-ablation --extra-workload none --workload bert_large --steps 10 > gpurun_out/gab_bertl_$lib.log 2>&1; echo "bench bertl rc=$?"
grep '"metric"' gpurun_out/gab_bertl_$lib.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['compute_only_ms'], d['roofline']['frac'], json.dumps(d['gemm_tiles']))"
done
