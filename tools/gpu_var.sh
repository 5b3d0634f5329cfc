for v in mb22 mb32 mb43; do
  for bps in 2 3 4; do
    RDMR_R4_BPS=$bps RDMR_LIB=build_variants/librdmr_$v.so timeout 300 python tools/strang_prof.py 3 4 > gpurun_out/var3_${v}_$bps.log 2>&1
    RDMR_R4_BPS=$bps RDMR_LIB=build_variants/librdmr_$v.so timeout 300 python tools/strang_prof.py 4 3 > gpurun_out/var4_${v}_$bps.log 2>&1
  done
done
