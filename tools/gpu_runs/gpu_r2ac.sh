nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2ac_gpu.txt
timeout 1500 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_nagumo.py -q -x > gpurun_out/r2ac_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ac_gpu.txt
for rep in 1 2; do for v in gold default; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2ac_c2_${v}_$rep.log 2>&1
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ac_c4_${v}_$rep.log 2>&1
done; done
