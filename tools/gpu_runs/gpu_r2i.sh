# profiles: radau5_thread (cfg 2 prefix), radau5_warp<20> (cfg 5), 3-D assembled-row stats, cfg 5 bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2i_gpu.txt
RDMR_R4_MODE=mat RDMR_MAT_DEBUG=1 timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2i_mat3d.log 2>&1; echo "mat3d rc=$?" >> gpurun_out/r2i_gpu.txt
timeout 300 python tools/r5_once.py 1048576 > gpurun_out/r2i_r5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -c 1 -o gpurun_out/r2i_r5c2 python tools/r5_once.py 1048576 > gpurun_out/r2i_r5_ncu.log 2>&1; echo "ncu r5 rc=$?" >> gpurun_out/r2i_gpu.txt
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2i_c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/r2i_gpu.txt
timeout 300 python tools/r5_cfg5.py > gpurun_out/r2i_r5w_plain.log 2>&1; echo "r5w rc=$?" >> gpurun_out/r2i_gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_warp -c 1 -o gpurun_out/r2i_r5w python tools/r5_cfg5.py > gpurun_out/r2i_r5w_ncu.log 2>&1; echo "ncu r5w rc=$?" >> gpurun_out/r2i_gpu.txt
