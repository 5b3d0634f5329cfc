# 3-D Rock4: simple projections done by the stage per chunk (no projection phase / barrier after round 0
# when every needed node is simple) vs HEAD; parity subset
for rep in 1 2; do for v in cur pchunk; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2ck_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_pchunk.so timeout 1500 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_two_point.py -q -x -k "rock4 or fv_apply or strang or cfg4 or adapt or two_point" > gpurun_out/r2ck_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2ck_tests.log
