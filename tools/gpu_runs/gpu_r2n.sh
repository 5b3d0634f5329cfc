# two-buffer Rock4 recurrence: Rock4 / Strang parity, r4_once cfg 4 / 3, benches cfg 4 / 3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2n_gpu.txt
timeout 1800 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_two_point.py tests/test_gpu_nagumo.py tests/test_gpu_max_sizes.py -q -x -k "not cfg5_full" > gpurun_out/r2n_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2n_gpu.txt
timeout 300 python tools/r4_once.py 4 3 > gpurun_out/r2n_r4c4.log 2>&1
timeout 300 python tools/r4_once.py 3 3 > gpurun_out/r2n_r4c3.log 2>&1
for c in 4 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n_c$c.log 2>&1; echo "c$c rc=$?" >> gpurun_out/r2n_gpu.txt; done
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_rock4 -c 2 --csv --log-file gpurun_out/r2n_r4_dram.csv python tools/r4_once.py 4 2 > gpurun_out/r2n_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2n_gpu.txt
