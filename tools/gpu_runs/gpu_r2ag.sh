# outlier hunt: default bench five times (per-step times in the JSON line)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ag_gpu.txt
for rep in 1 2 3 4 5; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2ag_b$rep.log 2>&1; done
