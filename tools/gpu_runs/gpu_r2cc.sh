# significance: skip the division for species scales s_i = 1 (div1) vs HEAD: adapt section profile cfg 4, bit-exact MR tests
for v in gold div1; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2cc_adapt4_$v.log 2>&1
done
RDMR_LIB=$PWD/build_variants/librdmr_div1.so timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "build or adapt or tie or calibration or cfg3 or cfg4 or degenerate" > gpurun_out/r2cc_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2cc_tests.log
