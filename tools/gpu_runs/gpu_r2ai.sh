nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ai_gpu.txt
timeout 1500 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_two_point.py -q -x -k "not cfg5_full and not cfg3_five and not cfg4_two" > gpurun_out/r2ai_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ai_gpu.txt
for rep in 1 2 3; do for v in gold default; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  timeout 300 python tools/r4_once.py 3 4 > gpurun_out/r2ai_r4c3_${v}_$rep.log 2>&1
  timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2ai_r4c4_${v}_$rep.log 2>&1
done; done
