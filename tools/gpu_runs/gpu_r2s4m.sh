# round 2 session 4: scheduling-key candidates timed with explicit orders (cfg 2 cells, cfg-4 half steps)
for w in cfg2 cfg4h1 cfg4h2; do timeout 600 python tools/r5_keys.py $w > gpurun_out/s4m_keys_$w.log 2>&1; echo "$w rc=$?"; cat gpurun_out/s4m_keys_$w.log; done
