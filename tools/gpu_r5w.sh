timeout 200 python tools/r5_cfg5.py > gpurun_out/r5_cfg5.log 2>&1
timeout 600 python -m pytest -q -x tests/test_gpu_radau5.py -k "mass_action or cfg5" > gpurun_out/r5w_t.log 2>&1
