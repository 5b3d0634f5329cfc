# operator build: one host read fewer (rho_1, level range and flags with the expansion count); GPU suite, bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2cg_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2cg_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2cg_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2cg_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2cg_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2cg_adapt4.log 2>&1
