python tools/r5_once.py 1048576 > gpurun_out/r5_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:radau5_thread -c 1 -o gpurun_out/r5_prof python tools/r5_once.py 1048576 > gpurun_out/r5_ncu.log 2>&1
echo done $?
