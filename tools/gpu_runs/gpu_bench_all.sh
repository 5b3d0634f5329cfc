# one bench line per config (no CPU baseline except where asked)
for c in 3 1 5 4 2; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 ${CPUB:---no-cpu-baseline} > gpurun_out/bench_c$c.log 2>&1
  echo "config $c rc=$?" >> gpurun_out/bench_rc.log
done
