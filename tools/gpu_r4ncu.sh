timeout 300 python -m pytest tests/test_gpu_mr_rock4.py -x -q -k "rock4 or strang" > gpurun_out/t_tests.log 2>&1; echo "exit $?" >> gpurun_out/t_tests.log
RDMR_LIB=build_variants/librdmr_t.so timeout 120 python tools/r4_mat_prof.py > gpurun_out/t_r4.log 2>&1
python tools/r4_mat_prof.py > gpurun_out/r4_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rock4_mat -s 1 -c 1 -o gpurun_out/r4matw32 python tools/r4_mat_prof.py > gpurun_out/r4_ncu.log 2>&1
