# 3-D Rock4 stage: species per row group 3 / 2 / 1
for rep in 1 2; do for v in sg3 sg2 sg1; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2by_r4c4_${v}_$rep.log 2>&1
done; done
