# 3-D Rock4 stage prefetch modes: 0 ticket ring only, 1 prefetch.global.L1, 2 prefetch.global.L2 (vs gold)
for rep in 1 2; do for v in gold pfm0 pfm1 pfm2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2bc_r4c4_${v}_$rep.log 2>&1
done; done
