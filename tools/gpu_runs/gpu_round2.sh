# round-1 (continued) measurement pass: GPU tests, smoke, default bench + configs, launch list and ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/r2_bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_ref.log 2>&1
for c in 1 2 4 5; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2_c$c.log 2>&1; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b2.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rock4_mat -s 2 -c 1 -o gpurun_out/r2_rock4mat python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 4 -c 1 -o gpurun_out/r2_radau5_cfg3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2_ncu3.log 2>&1
