# pool headroom at mr_grid_build: first steps after one restart (cfg 4, cfg 3), cfg 3 bench line
timeout 600 python tools/first_step.py 4 3 4 > gpurun_out/r2bw_c4.log 2>&1
timeout 600 python tools/first_step.py 3 3 4 > gpurun_out/r2bw_c3.log 2>&1
for c in 3 4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2bw_b$c.log 2>&1; done
