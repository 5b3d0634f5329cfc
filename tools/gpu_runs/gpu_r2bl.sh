# cfg 5 warp kernel: row-per-lane Gauss-Jordan in shared memory with implicit pivoting (row4: 16 warps/SM
# at 128 registers; row3: 12 warps at 168) vs the column-per-lane elimination with f3 (smem3)
for v in smem3 row4 row3; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python tools/r5w_time.py 65536 > gpurun_out/r2bl_${v}.log 2>&1
done
RDMR_LIB=$PWD/build_variants/librdmr_row4.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_mr_rock4.py -q -x -k "warp or cfg5 or mass or network" > gpurun_out/r2bl_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bl_tests.log
