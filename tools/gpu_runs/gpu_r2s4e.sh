# round 2 session 4: dump a cell sample (states before each half step, attempt counts) of cfg-4 steps for the cost-proxy study
R5_DUMP=gpurun_out/s4e_cells timeout 600 python tools/r5_halves.py 4 3 > gpurun_out/s4e_halves_c4.log 2>&1; echo rc=$?
ls -la gpurun_out/
