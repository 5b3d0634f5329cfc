python tools/r4_mat_prof.py > gpurun_out/r4_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rock4_mat -c 1 -o gpurun_out/r4matc python tools/r4_mat_prof.py > gpurun_out/r4_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4_launches.csv python tools/r4_mat_prof.py > gpurun_out/r4_ncu2.log 2>&1
