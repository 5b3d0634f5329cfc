"""Summarise bench JSON lines: python tools/blines.py LOG..."""
import json
import sys

for p in sys.argv[1:]:
    for ln in open(p):
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        r = d.get("roofline") or {}
        ph = r.get("phases")
        s = f"{p.split('/')[-1]:28s} {d['value']:.4g} {d['unit']:>20s} ms/step {d['ms_per_step']:.3f} e2e {d['e2e']['value']:.4g}"
        if ph:
            s += "  " + " ".join(f"{k}:{v['ms'] / d['steps']:.2f}ms/{v['frac']:.3f}" for k, v in ph.items())
        else:
            s += f"  frac {r.get('frac', 0):.3f}"
        print(s)
