for v in base l16 l12 base; do
  echo "== $v" >> gpurun_out/v_r4lane.log
  if [ $v = base ]; then timeout 120 python tools/r4_mat_prof.py >> gpurun_out/v_r4lane.log 2>&1
  else RDMR_LIB=build_variants/librdmr_$v.so timeout 120 python tools/r4_mat_prof.py >> gpurun_out/v_r4lane.log 2>&1; fi
done
