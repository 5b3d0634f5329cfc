python tools/r5w_once.py 32768 > gpurun_out/r5w_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:radau5_warp -c 1 -f -o gpurun_out/r5w_prof python tools/r5w_once.py 32768 > gpurun_out/r5w_ncu.log 2>&1
echo done $? >> gpurun_out/r5w_plain.log
