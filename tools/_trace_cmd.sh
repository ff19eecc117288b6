for mode in 1 0; do
for k in ff bp; do
  DEAR_GEMM_PAIR=$mode python tools/trace_gemm.py --workload resnet50 --kind $k --launches 4 | python3 -c "
import sys,json; d=json.loads(sys.stdin.read()); print('pair=$mode', d['kind'], {k:v for k,v in d['plans'].items()}); [print({k:(round(v,2) if isinstance(v,float) else v) for k,v in l.items()}) for l in d['launches'][1:]]"
done; done
python tools/gemm_cadence.py resnet_ff bertl_ff; DEAR_GEMM_PAIR=0 python tools/gemm_cadence.py resnet_ff bertl_ff
