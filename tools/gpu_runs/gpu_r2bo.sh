# cfg 5 warp kernel: elimination blocked by two pivot steps (b2) vs one step per pass (row3)
for v in row3 b2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python tools/r5w_time.py 65536 > gpurun_out/r2bo_${v}.log 2>&1
done
RDMR_LIB=$PWD/build_variants/librdmr_b2.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_mr_rock4.py -q -x -k "warp or cfg5 or mass or network" > gpurun_out/r2bo_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bo_tests.log
