for s in 4 8 12 16 20 24 32; do RDMR_R5_SCHED=$s timeout 300 python bench.py --config 2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s_$s.log 2>&1; done
