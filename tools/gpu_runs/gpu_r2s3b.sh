# round 2 session 3: ncu --set full of radau5_thread<3> on cfg 2 and radau5_warp<20> on cfg-5 cells (stall reasons, instruction mix)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 1 -c 1 -o gpurun_out/s3b_prof_r5 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s3b_ncu_r5.log 2>&1; echo "r5 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_warp -c 1 -o gpurun_out/s3b_prof_r5w python tools/r5w_once.py 32768 > gpurun_out/s3b_ncu_r5w.log 2>&1; echo "r5w rc=$?"
