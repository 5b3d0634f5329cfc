# full GPU test pass + a config-2 scheduling sweep
bash tools/gpu_tests.sh tests/test_gpu_mr_rock4.py tests/test_gpu_radau5.py -q > gpurun_out/t_all.log 2>&1
for s in 1 8 16 24; do RDMR_R5_SCHED=$s timeout 300 python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_s$s.log 2>&1; done
