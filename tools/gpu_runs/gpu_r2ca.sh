# current build: GPU suite, default bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ca_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2ca_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ca_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ca_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2ca_gpu.txt
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ca_c3.log 2>&1
