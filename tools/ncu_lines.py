"""Stall samples and executed instructions aggregated by CUDA source line of one kernel in an ncu report
(ncu --page source --print-source cuda,sass).  usage: python tools/ncu_lines.py REPORT [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg = {}
line = None
fname = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0] != "":
        line = (fname, int(r[0]), r[1].strip()[:90])
    if line is None or r[2] == "":
        continue
    try:
        s = int(r[4] or 0)
        ex = int(r[7] or 0)
    except ValueError:
        continue
    a = agg.setdefault(line, [0, 0])
    a[0] += s
    a[1] += ex
tot = sum(v[0] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100.0 * v[0] / tot:5.1f}%  {v[1]:>12}  {k[0]}:{k[1]}  {k[2]}")
