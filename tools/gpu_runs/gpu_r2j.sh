# full GPU suite; benches cfg 2/4/3/5/1; 1-core oracle per phase
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2j_gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2j_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2j_gpu.txt
for c in 2 4 3; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_c$c.log 2>&1; echo "c$c rc=$?" >> gpurun_out/r2j_gpu.txt; done
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/r2j_gpu.txt
timeout 600 python bench.py --config 1 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_c1.log 2>&1; echo "c1 rc=$?" >> gpurun_out/r2j_gpu.txt
timeout 600 python tools/r4_once.py 4 3 > gpurun_out/r2j_r4.log 2>&1; echo "r4 rc=$?" >> gpurun_out/r2j_gpu.txt
timeout 900 python tools/oracle_1core.py > gpurun_out/r2j_oracle_1core.json 2> gpurun_out/r2j_oracle_1core.err; echo "o1 rc=$?" >> gpurun_out/r2j_gpu.txt
