# Radau5 thread kernel: Oregonator f in FMA form (fmaf) vs HEAD: cfg 2 batch and cfg 4 R phase; radau5 parity
for rep in 1 2; do for v in gold fmaf; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2ci_c2_${v}_$rep.log 2>&1
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2ci_c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_fmaf.so timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_nagumo.py -q -x > gpurun_out/r2ci_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ci_tests.log
