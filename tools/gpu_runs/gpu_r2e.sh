# round 2 (session 2) evidence pass: GPU suite, smoke, default bench with cpu baseline, other configs,
# reference arm, launch list of the default bench, ncu --set full of k_rock4<3> / radau5_thread<3> (default
# bench) and radau5_warp<20> (32 768 cfg-5 cells)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2e_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2e_gpu.txt
for c in 2 3 1 5 6; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2e_c$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2e_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2e_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2e_adapt4.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2e_launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2e_ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -s 2 -c 1 -o gpurun_out/r2e_prof_rock4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2e_ncu_r4.log 2>&1; echo "full r4 rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 2 -c 1 -o gpurun_out/r2e_prof_radau5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2e_ncu_r5.log 2>&1; echo "full r5 rc=$?" >> gpurun_out/r2e_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:radau5_warp -c 1 -o gpurun_out/r2e_prof_r5w python tools/r5w_once.py 32768 > gpurun_out/r2e_ncu_r5w.log 2>&1; echo "full r5w rc=$?" >> gpurun_out/r2e_gpu.txt
