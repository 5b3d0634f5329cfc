# Radau5 thread kernel: two tickets per refill (tk2) vs HEAD: cfg 2 batch and cfg 4 bench R phase
for rep in 1 2; do for v in gold tk2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2cb_c2_${v}_$rep.log 2>&1
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2cb_c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_tk2.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_nagumo.py tests/test_gpu_shard.py -q -x > gpurun_out/r2cb_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2cb_tests.log
