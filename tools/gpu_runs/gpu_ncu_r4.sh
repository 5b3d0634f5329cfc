python tools/r4_once.py ${CFG:-4} 1 > gpurun_out/r4_plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -c 1 -o gpurun_out/r4_prof${CFG:-4} python tools/r4_once.py ${CFG:-4} 1 > gpurun_out/r4_ncu.log 2>&1
echo done $?
