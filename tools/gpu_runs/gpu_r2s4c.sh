# round 2 session 4: adaptation section times and Radau5 work statistics of cfg 4, ncu --set full of one cfg-4 Radau5 launch
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/s4c_adapt_c4.log 2>&1
timeout 300 python tools/r5_stats.py 4 4 > gpurun_out/s4c_stats_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 4 -c 1 -o gpurun_out/s4c_prof_r5c4 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/s4c_ncu_r5.log 2>&1; echo "r5 rc=$?"
tail -20 gpurun_out/s4c_stats_c4.log
