# Radau5 MINB=4 variant vs default on cfg 2 / 4; launch list of the default bench (cfg 4)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2k_gpu.txt
for v in default m4; do
  if [ $v = default ]; then unset RDMR_LIB; else export RDMR_LIB=$PWD/build_variants/librdmr_$v.so; fi
  timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_c2_$v.log 2>&1
  timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_c4_$v.log 2>&1
done
unset RDMR_LIB
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2k_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2k_launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2k_ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/r2k_gpu.txt
