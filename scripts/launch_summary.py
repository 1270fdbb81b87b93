"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel share of
the last `steps` steps (launches are cold-cache and serialised: compare shares)."""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
total_steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
data = [dict(zip(h, r)) for r in rows[hdr + 1:] if len(r) == len(h)]
seq = [(d["Kernel Name"].split("(")[0].replace("void ", "")[:58], float(d["Metric Value"]))
       for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
per_step = len(seq) // total_steps
last = seq[-per_step * steps:]
agg = collections.OrderedDict()
for nm, v in last:
    a = agg.setdefault(nm, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(v for v, _ in agg.values())
print(f"{len(seq)} launches, {per_step}/step; last {steps} steps: {tot/1e3/steps:.1f} us/step of kernel time")
for nm, (v, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {nm:58s} x{c // steps:<2d} {v / 1e3 / steps:9.1f} us/step {100 * v / tot:5.1f}%")
