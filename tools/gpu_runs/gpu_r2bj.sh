# ncu --set full of the cfg-5 warp kernel (f3 build), 16384 cells
RDMR_LIB=$PWD/build_variants/librdmr_f3.so timeout 1500 ncu --set full --clock-control none --import-source on -k regex:radau5_warp -c 1 -o gpurun_out/r2bj_prof_r5w python tools/r5w_time.py 16384 > gpurun_out/r2bj_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/r2bj_ncu.log
