# launch list (per-kernel device time) of the default bench command, then a full capture of k_rock4
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_plain.log 2>&1 &&
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_plain.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -s 2 -c 1 -o gpurun_out/prof_default_rock4 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_thread -s 2 -c 1 -o gpurun_out/prof_default_radau5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full_r5.log 2>&1
echo "full r5 rc=$?" >> gpurun_out/ncu_plain.log
