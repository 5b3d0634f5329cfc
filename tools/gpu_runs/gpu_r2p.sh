nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2p_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2p_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2p_gpu.txt
timeout 300 python tools/r4_once.py 4 3 > gpurun_out/r2p_r4c4.log 2>&1
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2p_r4t.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2p_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2p_gpu.txt
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_c3.log 2>&1
