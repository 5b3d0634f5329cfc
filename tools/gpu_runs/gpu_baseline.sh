# state-of-HEAD check: gpu tests, smoke, default bench, config 2 and 5 bench lines
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/hb_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/hb_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/hb_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/hb_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/hb_bench.log 2>&1
for c in 1 2 4 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/hb_c$c.log 2>&1; done
