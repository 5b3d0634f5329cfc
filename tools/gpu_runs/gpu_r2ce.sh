# 3-D Rock4: 128-row chunks / 10 blocks per SM (ch128) vs 256 / 5 (cur); per-phase round timing of cur
for rep in 1 2; do for v in cur ch128; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2ce_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_curt.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2ce_timing.log 2>&1
