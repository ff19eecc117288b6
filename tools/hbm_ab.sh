set -u
mkdir -p gpurun_out
for wl in resnet50 bert_large; do
for lib in ${LIBS:-libdear_old.so libdear.so libdear_s3.so libdear_s2.so libdear_s2u8.so}; do
DEAR_LIB=$lib timeout 300 python tools/hbm_chain.py --workload $wl 2>&1 | tail -1
done; done
