# cfg 5 warp kernel: elimination in registers, inverse rows in shared memory (rr2/rr3/rr4: 2/3/4 blocks of
# 4 warps per SM) vs row-per-lane shared-memory elimination (row3)
for v in row3 rr2 rr3 rr4; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python tools/r5w_time.py 65536 > gpurun_out/r2bn_${v}.log 2>&1
done
RDMR_LIB=$PWD/build_variants/librdmr_rr3.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_mr_rock4.py -q -x -k "warp or cfg5 or mass or network" > gpurun_out/r2bn_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bn_tests.log
