# 3-D Rock4: projection phase with 8 lanes per needed node (proj8) vs HEAD; per-phase round timing of both
for rep in 1 2; do for v in gold proj8; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2bs_r4c4_${v}_$rep.log 2>&1
done; done
for v in goldt proj8t; do RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2bs_timing_$v.log 2>&1; done
RDMR_LIB=$PWD/build_variants/librdmr_proj8.so timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "rock4 or fv_apply or strang_small_3d or cfg4" > gpurun_out/r2bs_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bs_tests.log
