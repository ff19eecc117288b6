#!/bin/bash
# A/B of GEMM library variants on one box: tools/ab_gemm.sh lib1 lib2 ...
for rep in 1 2; do
for lib in "$@"; do
  for w in resnet50 bert_large; do
    DEAR_LIB=$lib timeout 100 python tools/bench_gemm.py --workload $w --iters 100 | python3 -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['workload'], {k: round(d[k]['us'],2) for k in ('ff','dgrad','wgrad','bp_group')}, '8192', round(d['ours_8192']['tflops']))"
  done
done
done
