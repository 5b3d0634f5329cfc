# 3-D Rock4 stage: chunk prefetch (cp.async topology + own-row operands) vs HEAD (gold); parity of the variant
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2bb_gpu.txt
for rep in 1 2 3; do for v in gold pf; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2bb_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_pf.so timeout 1200 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "rock4 or fv_apply or strang_small_3d or cfg4" > gpurun_out/r2bb_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2bb_gpu.txt
