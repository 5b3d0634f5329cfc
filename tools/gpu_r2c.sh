# profiling pass: adapt sections on cfg 4/3, Radau5 scheduler sweep on cfg 2, ncu of k_rock4<3> (cfg 4)
# and radau5_thread<3> (cfg 2 prefix), then the new full-size parity tests
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2c_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2c_adapt4.log 2>&1; echo "adapt4 rc=$?" >> gpurun_out/r2c_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 3 > gpurun_out/r2c_adapt3.log 2>&1; echo "adapt3 rc=$?" >> gpurun_out/r2c_gpu.txt
for s in 8 16 20 28 32; do RDMR_R5_SCHED=$s timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/r2c_sched$s.log 2>&1; done
echo "sched done" >> gpurun_out/r2c_gpu.txt
timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2c_r4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -c 1 -o gpurun_out/r2c_r4c4 python tools/r4_once.py 4 1 > gpurun_out/r2c_r4_ncu.log 2>&1; echo "ncu r4 rc=$?" >> gpurun_out/r2c_gpu.txt
timeout 300 python tools/r5_once.py 1048576 > gpurun_out/r2c_r5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -c 1 -o gpurun_out/r2c_r5c2 python tools/r5_once.py 1048576 > gpurun_out/r2c_r5_ncu.log 2>&1; echo "ncu r5 rc=$?" >> gpurun_out/r2c_gpu.txt
timeout 2400 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "cfg3_five or cfg4_two or cfg5_full or tie or forced" --durations=10 > gpurun_out/r2c_fullsize.log 2>&1; echo "fullsize rc=$?" >> gpurun_out/r2c_gpu.txt
