# round 2 session 4: leaf keys + attempt counts of both half steps over consecutive cfg-4 steps (does the previous step's count predict this step's?)
R5_DUMPK=gpurun_out/s4g_keys timeout 600 python tools/r5_halves.py 4 4 > gpurun_out/s4g_halves_c4.log 2>&1; echo rc=$?
ls -la gpurun_out/
