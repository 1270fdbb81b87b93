"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: this framework's
kernels (namespace fssdp) of the last `steps` steps, `per_step` launches each.  ncu times
are cold-cache and serialised: compare SHARES of the step, not absolute step times.

    python scripts/launch_summary.py gpurun_out/launches.csv [steps=2] [per_step=15]
"""
import collections
import csv
import sys

path = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
per_step = int(sys.argv[3]) if len(sys.argv) > 3 else 15
OURS = ("gate_", "dispatch", "combine", "grouped_gemm", "spag", "sprs", "push_host",
        "pull_host", "barrier", "local_gemm", "route_scan", "adam", "epoch")


def _ours(name: str) -> bool:
    """This framework's kernels (ncu prints them with or without the fssdp:: namespace)."""
    base = name.replace("void ", "").replace("fssdp::", "").split("(")[0]
    return base.startswith(OURS) or "fssdp::" in name


rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
data = [dict(zip(h, r)) for r in rows[hdr + 1:] if len(r) == len(h)]
unit = data[0]["Metric Unit"] if data else "ns"
to_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}[unit]
seq = [(d["Kernel Name"].split("(")[0].replace("void ", "")[:58], float(d["Metric Value"]) * to_us)
       for d in data if d["Metric Name"] == "gpu__time_duration.sum" and _ours(d["Kernel Name"])]
last = seq[-per_step * steps:]
agg = collections.OrderedDict()
for nm, v in last:
    a = agg.setdefault(nm, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(v for v, _ in agg.values())
print(f"{len(seq)} fssdp launches; last {steps} steps x {per_step}: {tot / steps:.1f} us/step of kernel time")
for nm, (v, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"  {nm:58s} x{c // steps:<2d} {v / steps:9.1f} us/step {100 * v / tot:5.1f}%")
