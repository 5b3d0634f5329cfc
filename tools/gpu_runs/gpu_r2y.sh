# A/B: host-driven fixed points (gold = previous commit) vs cooperative fixed points (default)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2y_gpu.txt
for rep in 1 2; do for v in gold default; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  for c in 3 4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2y_c${c}_${v}_$rep.log 2>&1; done
done; done
