"""Summarises an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel share of device time."""
import collections
import csv
import re
import sys


def summarise(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    t, c = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik]
        name = re.sub(r"^void ", "", name)
        name = re.sub(r"\(.*", "", name)          # drop the argument list
        name = name.replace("<unnamed>::", "")
        name = re.sub(r"<.*", lambda m: "<" + m.group(0)[1:].split(",")[0].split(">")[0] + ">", name)
        v = float(r[iv].replace(",", ""))
        v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[iu], 1e-6)
        t[name] += v
        c[name] += 1
    tot = sum(t.values())
    out = [f"total device time {tot:.3f} ms over {sum(c.values())} launches (cold-cache, serialised by ncu)"]
    for k, v in t.most_common(top):
        out.append(f"{100 * v / tot:6.2f}%  {v:9.3f} ms  n={c[k]:4d}  {k}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
