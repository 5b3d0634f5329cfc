# round 2 (session 4) evidence pass: GPU suite, smoke, default bench with cpu baseline, other configs,
# reference arm, launch list of the default bench, ncu --set full of k_rock4<3> / radau5_thread<3> (default bench)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2f_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 900 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 900 python bench.py > gpurun_out/r2f_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2f_gpu.txt
for c in 2 3 1 5 6; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_c$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2f_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2f_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2f_adapt4.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2f_launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2f_ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -s 2 -c 1 -o gpurun_out/r2f_prof_rock4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2f_ncu_r4.log 2>&1; echo "full r4 rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 3 -c 1 -o gpurun_out/r2f_prof_radau5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2f_ncu_r5.log 2>&1; echo "full r5 rc=$?" >> gpurun_out/r2f_gpu.txt
cat gpurun_out/r2f_gpu.txt; tail -3 gpurun_out/r2f_tests.log
python tools/blines.py gpurun_out/r2f_bench_default.log gpurun_out/r2f_c*.log
