# round 2 session 4: default bench at 20 steps / 5 warm-up (the window of profiles/r02b_bench_default_cfg4.json), three repetitions
for rep in 1 2 3; do timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/s4q_c4_20_$rep.log 2>&1; done
python tools/blines.py gpurun_out/s4q_c4_20_*.log
