nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2s_gpu.txt
timeout 300 python tools/grid_stats.py > gpurun_out/r2s_stats.log 2>&1; echo "stats rc=$?" >> gpurun_out/r2s_gpu.txt
