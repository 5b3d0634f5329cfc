# 3-D Rock4: ghost phase with inline projections (no projection phase / barrier) vs HEAD
for rep in 1 2; do for v in gold ginl; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2br_r4c4_${v}_$rep.log 2>&1
done; done
