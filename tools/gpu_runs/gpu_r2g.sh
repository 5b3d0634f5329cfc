# full GPU suite (+ the 2-rank shard test), benches cfg 2 / 4 / 3, adapt profile cfg 4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2g_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu --durations=8 > gpurun_out/r2g_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2g_gpu.txt
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_c2.log 2>&1; echo "c2 rc=$?" >> gpurun_out/r2g_gpu.txt
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/r2g_gpu.txt
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_c3.log 2>&1; echo "c3 rc=$?" >> gpurun_out/r2g_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2g_adapt4.log 2>&1; echo "adapt4 rc=$?" >> gpurun_out/r2g_gpu.txt
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2g_r4t.log 2>&1; echo "r4t rc=$?" >> gpurun_out/r2g_gpu.txt
