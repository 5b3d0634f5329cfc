# 3-D Rock4: same-level gathers issued unconditionally (nbu), + projection expansions in batches of 4 (nbup)
for rep in 1 2; do for v in gold nbu nbup; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2bg_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_nbup.so timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "rock4 or fv_apply or strang_small_3d or cfg4" > gpurun_out/r2bg_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bg_tests.log
