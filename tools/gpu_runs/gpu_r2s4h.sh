# round 2 session 4: full GPU suite on the proxy-LPT build (65536-cell gate), event-trip threshold sweep on cfg 4 / cfg 2, cfg 1 check
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/s4h_tests.log 2>&1; echo "tests rc=$?"
for s in 12 16 20 24 28; do
  RDMR_R5_SCHED=$s timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4h_c4_s$s.log 2>&1
  RDMR_R5_SCHED=$s timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s4h_c2_s$s.log 2>&1
done
timeout 300 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/s4h_c1.log 2>&1
tail -3 gpurun_out/s4h_tests.log
python tools/blines.py gpurun_out/s4h_c*.log
