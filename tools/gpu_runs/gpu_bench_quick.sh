for c in 3 4 5; do timeout 900 python bench.py --config $c --steps ${STEPS:-3} --warmup 1 --no-cpu-baseline > gpurun_out/q_c$c.log 2>&1; done
