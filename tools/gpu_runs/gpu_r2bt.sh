# one-off costs of the first steps after bench.py's restart (cfg 4 and cfg 6)
timeout 600 python tools/first_step.py 4 3 4 > gpurun_out/r2bt_c4.log 2>&1
timeout 600 python tools/first_step.py 6 3 4 > gpurun_out/r2bt_c6.log 2>&1
