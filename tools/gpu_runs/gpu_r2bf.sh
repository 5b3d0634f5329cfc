# 3-D Rock4 stage: warp tickets (no block barrier per chunk) vs HEAD
for rep in 1 2; do for v in gold wt1; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2bf_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_wt1.so timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "rock4 or fv_apply or strang_small_3d or cfg4" > gpurun_out/r2bf_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bf_tests.log
