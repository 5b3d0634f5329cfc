# round 2 session 4: final check of the committed tree: smoke, GPU suite, the driver's bench command
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4z_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/s4z_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4z_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/s4z_smoke.log; tail -2 gpurun_out/s4z_tests.log; python tools/blines.py gpurun_out/s4z_bench.log
