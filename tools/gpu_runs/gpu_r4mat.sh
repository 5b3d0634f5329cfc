# Rock4 assembled-operator check: rock4 + strang GPU tests, default bench (cfg 3), config 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/m_smi.txt
timeout 900 python -m pytest tests/test_gpu_mr_rock4.py -x -q -k "rock4 or strang" > gpurun_out/m_tests.log 2>&1; echo "exit $?" >> gpurun_out/m_tests.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench.log 2>&1
RDMR_R4_MODE=free timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_free.log 2>&1
timeout 300 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m_c1.log 2>&1
