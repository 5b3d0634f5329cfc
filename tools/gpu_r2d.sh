# 3-D Rock4 static rows: parity (Rock4 / Strang tests), timing cfg 4 / 3, launch list of cfg-4 adapts
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2d_gpu.txt
timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "not cfg5_full and not cfg3_five and not cfg4_two" > gpurun_out/r2d_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2d_gpu.txt
timeout 300 python tools/r4_once.py 4 3 > gpurun_out/r2d_r4.log 2>&1; echo "r4 rc=$?" >> gpurun_out/r2d_gpu.txt
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/r2d_gpu.txt
timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_c3.log 2>&1; echo "c3 rc=$?" >> gpurun_out/r2d_gpu.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_adapt_launches.csv python tools/adapt_prof.py 4 > gpurun_out/r2d_ncu_adapt.log 2>&1; echo "ncu adapt rc=$?" >> gpurun_out/r2d_gpu.txt
