# round 2, session 2: re-validate the restored HEAD (GPU suite, smoke, default bench, cfg 2 / 5 lines)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ba_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2ba_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2ba_gpu.txt
for c in 2 5; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ba_c$c.log 2>&1; done
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2ba_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ba_gpu.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ba_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2ba_gpu.txt
