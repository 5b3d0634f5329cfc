# round 2 session 3: Radau5 thread-kernel variants (split FP32 norm chains, live-lane event threshold), A/B on one box
for rep in 1 2; do
for v in base sa rs sars; do
  RDMR_LIB=build_variants/librdmr_$v.so timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3c_c2_${v}_$rep.log 2>&1
  RDMR_LIB=build_variants/librdmr_$v.so timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3c_c4_${v}_$rep.log 2>&1
done; done
for s in 20 28; do
  RDMR_R5_SCHED=$s RDMR_LIB=build_variants/librdmr_sars.so timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s3c_c2_sars_s$s.log 2>&1
  RDMR_R5_SCHED=$s RDMR_LIB=build_variants/librdmr_sars.so timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s3c_c4_sars_s$s.log 2>&1
done
RDMR_LIB=build_variants/librdmr_sars.so timeout 900 python -m pytest tests/test_gpu_radau5.py -q -x > gpurun_out/s3c_t_sars.log 2>&1; echo "tests rc=$?" >> gpurun_out/s3c_t_sars.log
python tools/blines.py gpurun_out/s3c_c*.log
