nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2x_gpu.txt
timeout 1800 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_max_sizes.py tests/test_gpu_nagumo.py tests/test_gpu_two_point.py tests/test_gpu_shard.py -q -x -k "not cfg5_full" > gpurun_out/r2x_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2x_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2x_adapt4.log 2>&1
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 3 > gpurun_out/r2x_adapt3.log 2>&1
for c in 4 3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2x_c$c.log 2>&1; done
