# round 2 (session 4) re-entry check: GPU suite, smoke, default bench, cfg 2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/s4a_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/s4a_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4a_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4a_gpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s4a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/s4a_gpu.txt
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4a_c2.log 2>&1
cat gpurun_out/s4a_gpu.txt; tail -3 gpurun_out/s4a_tests.log
