timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t_tests.log 2>&1; echo "exit $?" >> gpurun_out/t_tests.log
timeout 120 python tools/r4_mat_prof.py > gpurun_out/t_r4.log 2>&1
RDMR_LIB=build_variants/librdmr_t.so timeout 120 python tools/r4_mat_prof.py >> gpurun_out/t_r4.log 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t_bench.log 2>&1
