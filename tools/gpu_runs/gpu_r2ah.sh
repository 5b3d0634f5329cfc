nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ah_gpu.txt
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r2ah_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ah_gpu.txt
for rep in 1 2; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ah_b$rep.log 2>&1; done
