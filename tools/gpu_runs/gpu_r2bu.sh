# Rock4 warm start (h0 = the previous D call's proposal) vs HEAD: 6 consecutive D calls on cfg 4 / cfg 3
for v in gold warm; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 6 > gpurun_out/r2bu_r4c4_${v}.log 2>&1
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 3 6 > gpurun_out/r2bu_r4c3_${v}.log 2>&1
done
