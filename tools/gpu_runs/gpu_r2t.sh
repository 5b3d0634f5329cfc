nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2t_gpu.txt
timeout 1500 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_max_sizes.py -q -x -k "not cfg5_full and not cfg3_five" > gpurun_out/r2t_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2t_gpu.txt
for v in gold default gu3 gu9; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2t_r4_$v.log 2>&1
done
unset RDMR_LIB
