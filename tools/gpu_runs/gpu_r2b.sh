# radau5 thread-kernel variants: parity tests on the default build, cfg 2 / cfg 4 timings per variant
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2b_gpu.txt
timeout 900 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_nagumo.py -q -x > gpurun_out/r2b_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2b_gpu.txt
for v in default m4 m5; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_c2_$v.log 2>&1; echo "c2 $v rc=$?" >> gpurun_out/r2b_gpu.txt
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_c4_$v.log 2>&1; echo "c4 $v rc=$?" >> gpurun_out/r2b_gpu.txt
done
