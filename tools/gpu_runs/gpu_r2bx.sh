# 3-D Rock4 ghost phase: one (record, species) pair per thread (gsplit) vs HEAD
for rep in 1 2; do for v in gold gsplit; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2bx_r4c4_${v}_$rep.log 2>&1
done; done
