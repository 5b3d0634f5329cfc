# 3-D Rock4: per-chunk projections incl. chunk-straddling nodes (countdown), no projection phase after
# round 0 when every needed node's expansion is its 8 children (pchunk3) vs HEAD (cur); parity subset
for rep in 1 2; do for v in cur pchunk3; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2cm_r4c4_${v}_$rep.log 2>&1
done; done
RDMR_LIB=$PWD/build_variants/librdmr_pchunk3.so timeout 1500 python -m pytest tests/test_gpu_mr_rock4.py tests/test_gpu_two_point.py tests/test_gpu_shard.py -q -x -k "rock4 or fv_apply or strang or cfg4 or adapt or two_point or shard" > gpurun_out/r2cm_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2cm_tests.log
