# round 2 session 4: event-trip threshold with the 31-bit scheduling key
for s in 20 24 26 28 30; do
  RDMR_R5_SCHED=$s timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4o_c4_s$s.log 2>&1
  RDMR_R5_SCHED=$s timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4o_c2_s$s.log 2>&1
done
python tools/blines.py gpurun_out/s4o_c*.log
