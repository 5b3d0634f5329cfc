for b in 2 3 4; do RDMR_LIB=build_variants/librdmr_minb$b.so timeout 300 python bench.py --config 2 --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/r5v_$b.log 2>&1; done
