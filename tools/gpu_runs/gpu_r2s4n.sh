# round 2 session 4: previous step's per-cell work carried through the adaptation as the scheduling key (cfg 4, explicit orders)
timeout 900 python tools/r5_hist.py 4 5 > gpurun_out/s4n_hist_c4.log 2>&1; echo rc=$?
cat gpurun_out/s4n_hist_c4.log
