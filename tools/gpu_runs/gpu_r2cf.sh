# 3-D Rock4 ghost phase over a compact list of the type-2 records (if2) vs HEAD (cur); parity subset
for rep in 1 2; do for v in cur if2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2cf_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_if2.so timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "rock4 or fv_apply or strang_small_3d or cfg4 or adapt" > gpurun_out/r2cf_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2cf_tests.log
