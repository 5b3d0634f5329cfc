# current build: GPU suite, default bench (cfg 4), cfg 5 / cfg 2 lines
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2bp_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2bp_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2bp_gpu.txt
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2bp_c5.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2bp_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bp_gpu.txt
