# per-chunk projections of the simple nodes (pchunk2, the build) vs cur: A/B, GPU suite, default bench
for rep in 1 2; do for v in cur pchunk2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2cn_r4c4_${v}_$rep.log 2>&1
done; done
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2cn_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2cn_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2cn_bench_default.log 2>&1
