# round 2 session 4: how often is the first timed step of the cfg-4 bench slow (21-26 ms instead of 9.5), and which host call waits
for rep in 1 2 3 4 5 6 7 8 9 10 11 12; do
  RDMR_LIB=$PWD/build_variants/librdmr_trace.so timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4i_c4_$rep.log 2>&1
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/s4i_c4_*.log')):
    t=open(f).read(); l=[x for x in t.splitlines() if x.startswith('{')][-1]; d=json.loads(l)
    tr=[x for x in t.splitlines() if x.startswith('[trace]')]
    print(f, d['step_ms'], d['roofline']['phase_ms'], len(tr), tr[-6:])
PY
