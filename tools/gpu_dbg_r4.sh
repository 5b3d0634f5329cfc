timeout 60 python tools/r4_once.py 3 3 > gpurun_out/dbg_c3.log 2>&1
timeout 60 python tools/r4_once.py 1 3 > gpurun_out/dbg_c1.log 2>&1
timeout 100 python tools/r4_once.py 4 2 > gpurun_out/dbg_c4.log 2>&1
timeout 100 python tools/r4_once.py 5 2 > gpurun_out/dbg_c5.log 2>&1
timeout 200 python tools/adapt_prof.py 3 > gpurun_out/dbg_a3.log 2>&1
timeout 900 python -m pytest -q -x tests/test_gpu_mr_rock4.py -k "not table" > gpurun_out/dbg_t.log 2>&1
