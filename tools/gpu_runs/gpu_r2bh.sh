# 3-D Rock4 (nbup build): per-phase round timing (block 0) and one ncu --set full capture with source lines
RDMR_LIB=$PWD/build_variants/librdmr_nbupt.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2bh_timing.log 2>&1
RDMR_LIB=$PWD/build_variants/librdmr_nbup.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_rock4 -s 1 -c 1 -o gpurun_out/r2bh_prof_r4 python tools/r4_once.py 4 2 > gpurun_out/r2bh_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2bh_ncu.log
