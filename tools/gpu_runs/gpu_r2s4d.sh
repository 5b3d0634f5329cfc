# round 2 session 4: the two reaction half steps of a cfg-4 Strang step: work, time, and the LPT order's share
timeout 600 python tools/r5_halves.py 4 > gpurun_out/s4d_halves_c4.log 2>&1; echo rc=$?
cat gpurun_out/s4d_halves_c4.log
