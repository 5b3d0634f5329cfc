nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2w_gpu.txt
timeout 1800 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_max_sizes.py tests/test_gpu_two_point.py -q -x -k "not cfg5_full" > gpurun_out/r2w_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2w_gpu.txt
for rep in 1 2; do for v in gold default; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2w_r4_${v}_$rep.log 2>&1
done; done
unset RDMR_LIB
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2w_r4t.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2w_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2w_gpu.txt
