# round 2 session 4: Radau5 thread kernel, f / Newton counters updated per attempt (cnt) vs per iteration (base)
RDMR_LIB=$PWD/build_variants/librdmr_cnt.so timeout 900 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_nagumo.py -q -x > gpurun_out/s4p_t_cnt.log 2>&1; echo "tests rc=$?" >> gpurun_out/s4p_t_cnt.log
for rep in 1 2; do
for v in base cnt; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4p_c2_${v}_$rep.log 2>&1
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4p_c4_${v}_$rep.log 2>&1
done; done
tail -3 gpurun_out/s4p_t_cnt.log
python tools/blines.py gpurun_out/s4p_c*.log
