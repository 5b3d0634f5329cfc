# round-2 evidence pass 2 (current build): GPU suite, smoke, default bench with cpu baseline, other
# configs, launch list + ncu --set full of the two dominant kernels of the default bench, adapt profile,
# Rock4 timing split
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2v_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2v_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2v_gpu.txt
timeout 900 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2v_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2v_bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2v_gpu.txt
for c in 2 3 1 5 6; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2v_c$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2v_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/r2v_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2v_adapt4.log 2>&1
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2v_r4t.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2v_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2v_launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2v_ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2v_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -s 2 -c 1 -o gpurun_out/r2v_prof_rock4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2v_ncu_r4.log 2>&1; echo "full r4 rc=$?" >> gpurun_out/r2v_gpu.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 2 -c 1 -o gpurun_out/r2v_prof_radau5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2v_ncu_r5.log 2>&1; echo "full r5 rc=$?" >> gpurun_out/r2v_gpu.txt
