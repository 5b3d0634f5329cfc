# MR adapt changes: bit-exact MR tests + Strang parity, adapt section profile cfg 4 / 3, bench cfg 4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2e_gpu.txt
timeout 1500 python -m pytest tests -q -x -m gpu -k "not cfg5_full and not cfg4_two" > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2e_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2e_adapt4.log 2>&1; echo "adapt4 rc=$?" >> gpurun_out/r2e_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 3 > gpurun_out/r2e_adapt3.log 2>&1; echo "adapt3 rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_c3.log 2>&1; echo "c3 rc=$?" >> gpurun_out/r2e_gpu.txt
