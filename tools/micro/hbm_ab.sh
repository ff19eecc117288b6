# A/B of bucket-kernel grid / unroll build variants (tools/micro/hbm_stage.py).
for rep in 1 2; do
  for lib in libdear.so libdear_p3u8.so libdear_p2u8.so libdear_p3u5.so libdear_p4u5.so; do
    DEAR_LIB=$lib timeout 300 python tools/micro/hbm_stage.py 2>&1 | grep "^{"
  done
done
