nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2r_gpu.txt
timeout 1800 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_two_point.py tests/test_gpu_max_sizes.py tests/test_gpu_nagumo.py -q -x -k "not cfg5_full" > gpurun_out/r2r_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2r_gpu.txt
timeout 300 python tools/r4_once.py 4 3 > gpurun_out/r2r_r4c4.log 2>&1
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2r_r4t.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2r_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2r_gpu.txt
