# round 2 session 4: cfg 5 (m = 20, warp kernel): cell cost spread and the ideal longest-first order
timeout 600 python tools/r5w_order.py > gpurun_out/s4j_r5w_order.log 2>&1; echo rc=$?
cat gpurun_out/s4j_r5w_order.log
