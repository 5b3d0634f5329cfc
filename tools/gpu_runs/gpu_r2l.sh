# coarsening with blocked marks: bit-exact MR / Strang tests, adapt profiles, cfg 4 / 3 benches
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2l_gpu.txt
timeout 1800 python -m pytest tests -q -x -m gpu -k "not cfg5_full" > gpurun_out/r2l_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2l_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2l_adapt4.log 2>&1
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 3 > gpurun_out/r2l_adapt3.log 2>&1
for c in 4 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_c$c.log 2>&1; echo "c$c rc=$?" >> gpurun_out/r2l_gpu.txt; done
