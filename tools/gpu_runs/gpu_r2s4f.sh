# round 2 session 4: cost-proxy LPT order for every reaction substep (second half step, DRD, plain ABI call): tests + benches
timeout 1200 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_shard.py tests/test_gpu_mr_rock4.py tests/test_gpu_nagumo.py -q -x > gpurun_out/s4f_tests.log 2>&1; echo "tests rc=$?"
for c in 4 2 3 1; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4f_c$c.log 2>&1
  RDMR_NO_PROXY_LPT=1 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4f_c${c}_nolpt.log 2>&1
done
tail -3 gpurun_out/s4f_tests.log
python tools/blines.py gpurun_out/s4f_c*.log
