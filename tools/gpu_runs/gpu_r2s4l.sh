# round 2 session 4: 31-bit scheduling key (proxy, then the state's log-magnitudes) vs the 16-bit cost key (RDMR_LPT_KEY16=1)
timeout 600 python -m pytest tests/test_gpu_radau5.py tests/test_gpu_shard.py -q -x > gpurun_out/s4l_tests.log 2>&1; echo "tests rc=$?"
for rep in 1 2; do
for c in 4 3 2; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4l_c${c}_k31_$rep.log 2>&1
  RDMR_LPT_KEY16=1 timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4l_c${c}_k16_$rep.log 2>&1
done; done
tail -3 gpurun_out/s4l_tests.log
python tools/blines.py gpurun_out/s4l_c*.log
