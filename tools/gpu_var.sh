for v in inl0 inl1; do RDMR_LIB=build_variants/librdmr_$v.so timeout 100 python tools/r4_once.py 3 3 > gpurun_out/var_$v.log 2>&1; RDMR_LIB=build_variants/librdmr_$v.so timeout 100 python tools/r4_once.py 4 2 > gpurun_out/var4_$v.log 2>&1; done
RDMR_LIB=build_variants/librdmr_inl1.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/var_bench_inl1.log 2>&1
timeout 200 python tools/r5_cfg5.py > gpurun_out/r5_cfg5.log 2>&1
