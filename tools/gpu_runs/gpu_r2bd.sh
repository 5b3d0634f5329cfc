# 3-D Rock4 ticket order: 0 longest-first (HEAD), 1 heavy chunks longest-first + serpentine light chunks, 2 pure serpentine
for rep in 1 2; do for v in gold serp0 serp1 serp2; do
  RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 4 > gpurun_out/r2bd_r4c4_${v}_$rep.log 2>&1
done; done
