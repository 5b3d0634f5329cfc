# Radau5 per-kind specialisation: Radau5 tests, cfg 2 / 4 timing; adapt launch list on cfg 4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2f_gpu.txt
timeout 900 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_nagumo.py tests/test_gpu_shard.py -q -x > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_c2.log 2>&1; echo "c2 rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_adapt_launches.csv python tools/adapt_prof.py 4 > gpurun_out/r2f_ncu_adapt.log 2>&1; echo "ncu adapt rc=$?" >> gpurun_out/r2f_gpu.txt
timeout 300 python tools/r5_once.py 1048576 > gpurun_out/r2f_r5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -c 1 -o gpurun_out/r2f_r5c2 python tools/r5_once.py 1048576 > gpurun_out/r2f_r5_ncu.log 2>&1; echo "ncu r5 rc=$?" >> gpurun_out/r2f_gpu.txt
