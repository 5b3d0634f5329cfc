for v in base w48 w48g2 w32x2g1; do
  echo "== $v" >> gpurun_out/v_r4occ.log
  if [ $v = base ]; then timeout 120 python tools/r4_mat_prof.py >> gpurun_out/v_r4occ.log 2>&1
  else RDMR_LIB=build_variants/librdmr_$v.so timeout 120 python tools/r4_mat_prof.py >> gpurun_out/v_r4occ.log 2>&1; fi
done
