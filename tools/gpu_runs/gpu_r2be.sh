# cfg 5 warp-kernel counters per half step (jac / lu / newton mix) on the initial field
nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader > gpurun_out/r2be_gpu.txt
timeout 600 python tools/r5_cfg5.py > gpurun_out/r2be_cfg5.log 2>&1
