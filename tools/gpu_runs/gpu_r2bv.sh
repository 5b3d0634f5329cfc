# Rock4 warm start: GPU suite, default bench, cfg 3 / cfg 6 lines
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2bv_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2bv_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bv_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2bv_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2bv_gpu.txt
for c in 3 6 1; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2bv_c$c.log 2>&1; done
