# 3-D Rock4: 512-row chunks / 2 blocks of 512 per SM (ch512) vs 256 / 5 (cur)
for rep in 1 2; do for v in cur ch512; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2ch_r4c4_${v}_$rep.log 2>&1
done; done
