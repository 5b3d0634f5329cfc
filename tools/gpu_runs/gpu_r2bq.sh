# mr_adapt section profile on cfg 4 and cfg 3; launch list of the default bench
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2bq_adapt4.log 2>&1
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 3 > gpurun_out/r2bq_adapt3.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2bq_launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2bq_ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2bq_ncu_launch.log
