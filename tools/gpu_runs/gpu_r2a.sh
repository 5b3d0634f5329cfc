# round 2, first pass: GPU tests, smoke, forced-step rounding probe, bench cfg 4 (default) / 3 / 2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2a_gpu.txt
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_gpu.txt
timeout 300 python tools/r4_forced_err.py > gpurun_out/r2a_forced.log 2>&1; echo "forced rc=$?" >> gpurun_out/r2a_gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/r2a_gpu.txt
for c in 3 2; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_c$c.log 2>&1; echo "bench c$c rc=$?" >> gpurun_out/r2a_gpu.txt; done
