# Radau5 scheduler threshold and first-half-step ordering on cfg 4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2z_gpu.txt
for s in 24 16 20 28; do RDMR_R5_SCHED=$s timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_sched$s.log 2>&1; done
RDMR_NO_PROXY_LPT=1 timeout 900 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2z_nolpt.log 2>&1
