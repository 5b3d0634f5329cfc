timeout 600 python -m pytest tests/test_gpu_radau5.py -x -q > gpurun_out/t_tests.log 2>&1; echo "exit $?" >> gpurun_out/t_tests.log
timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v_c5_base.log 2>&1
RDMR_LIB=build_variants/librdmr_w4.so timeout 600 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/v_c5_w4.log 2>&1
