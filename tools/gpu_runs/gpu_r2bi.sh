# cfg 5 warp kernel: three stage f evaluations interleaved (f3) vs HEAD (gold)
for v in gold f3; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python tools/r5w_time.py 65536 > gpurun_out/r2bi_${v}.log 2>&1
done
RDMR_LIB=$PWD/build_variants/librdmr_f3.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_mr_rock4.py -q -x -k "warp or cfg5 or mass or network" > gpurun_out/r2bi_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bi_tests.log
