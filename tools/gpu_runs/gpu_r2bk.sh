# cfg 5 warp kernel: register-resident Gauss-Jordan (reg2: 255 regs / 8 warps per SM; reg3: 170 regs / 12 warps)
# vs the shared-memory kernel with f3 (smem3) and HEAD (gold)
for v in gold smem3 reg2 reg3; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python tools/r5w_time.py 65536 > gpurun_out/r2bk_${v}.log 2>&1
done
RDMR_LIB=$PWD/build_variants/librdmr_reg2.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_mr_rock4.py -q -x -k "warp or cfg5 or mass or network" > gpurun_out/r2bk_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bk_tests.log
