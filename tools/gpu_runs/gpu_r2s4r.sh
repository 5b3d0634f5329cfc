# round 2 session 4: scheduling keys of 16 / 24 / 31 bits (2 / 3 / 4 radix passes) timed with explicit orders
for w in cfg2 cfg4h1 cfg4h2; do timeout 600 python tools/r5_keys.py $w bits > gpurun_out/s4r_bits_$w.log 2>&1; echo "$w rc=$?"; cat gpurun_out/s4r_bits_$w.log; done
