nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2aa_gpu.txt
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 3 2 > gpurun_out/r2aa_r4t_c3.log 2>&1
RDMR_LIB=$PWD/build_variants/librdmr_r4t.so timeout 300 python tools/r4_once.py 4 2 > gpurun_out/r2aa_r4t_c4.log 2>&1
timeout 300 python tools/r4_once.py 3 3 > gpurun_out/r2aa_r4_c3.log 2>&1
