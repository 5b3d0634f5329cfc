# full GPU test suite, smoke, one bench line per config (cfg 3 with the CPU baseline)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/full_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/full_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/full_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full_gpu.txt
timeout 900 python bench.py > gpurun_out/full_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/full_gpu.txt
for c in 1 2 4 5 6; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/full_bench_c$c.log 2>&1; echo "bench c$c rc=$?" >> gpurun_out/full_gpu.txt; done
