timeout 600 python -m pytest tests/test_gpu_radau5.py -x -q > gpurun_out/t_tests.log 2>&1; echo "exit $?" >> gpurun_out/t_tests.log
for v in base mb4; do
  if [ $v = base ]; then L=""; else L="RDMR_LIB=build_variants/librdmr_$v.so"; fi
  env $L timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/v_c2_$v.log 2>&1
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/v_c3_$v.log 2>&1
done
