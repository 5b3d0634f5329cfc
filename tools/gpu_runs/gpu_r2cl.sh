# 3-D Rock4 per-chunk projections with (node, first leaf) list entries (pchunk2) vs HEAD (cur)
for rep in 1 2; do for v in cur pchunk2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2cl_r4c4_${v}_$rep.log 2>&1
done; done
