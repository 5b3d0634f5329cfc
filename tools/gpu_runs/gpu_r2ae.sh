nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ae_gpu.txt
timeout 1800 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_max_sizes.py tests/test_gpu_nagumo.py tests/test_gpu_shard.py -q -x -k "not cfg5_full" > gpurun_out/r2ae_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ae_gpu.txt
RDMR_ADAPT_PROFILE=1 timeout 300 python tools/adapt_prof.py 4 > gpurun_out/r2ae_adapt4.log 2>&1
for rep in 1 2; do for v in gold default; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  for c in 4 3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ae_c${c}_${v}_$rep.log 2>&1; done
done; done
