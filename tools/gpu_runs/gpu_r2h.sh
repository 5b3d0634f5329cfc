# 3-D Rock4: last-block error norm, ticket sweep, timing breakdown, 3-D assembled-row statistics
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r2h_gpu.txt
timeout 900 python -m pytest tests/test_gpu_mr_rock4.py -q -x -k "not cfg5_full and not cfg3_five" > gpurun_out/r2h_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2h_gpu.txt
for tc in 1 2 3; do RDMR_R4_TC=$tc timeout 300 python tools/r4_once.py 4 3 > gpurun_out/r2h_tc$tc.log 2>&1; done
for b in 3 5; do RDMR_R4_BPS=$b timeout 300 python tools/r4_once.py 4 3 > gpurun_out/r2h_bps$b.log 2>&1; done
RDMR_R4_MODE=mat RDMR_MAT_DEBUG=1 timeout 300 python tools/r4_once.py 4 1 > gpurun_out/r2h_mat3d.log 2>&1; echo "mat3d rc=$?" >> gpurun_out/r2h_gpu.txt
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2h_c4.log 2>&1; echo "c4 rc=$?" >> gpurun_out/r2h_gpu.txt
