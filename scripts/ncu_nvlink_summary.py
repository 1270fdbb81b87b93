"""Summarise an ncu --csv launch list with NVLink counters (scripts/nvlink_layer.py):
per kernel family and device, the LAST iteration's launches: time, NVLink user bytes in /
out, GB/s (user bytes ÷ kernel time), and raw link bytes (incl. protocol).

    python scripts/ncu_nvlink_summary.py gpurun_out/nvl_layer4_ncu.csv
"""

import argparse
import collections
import csv
import json
import re


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    col = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Device", "Metric Name", "Metric Value")}
    launches = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = int(r[col["ID"]])
        ent = launches.setdefault(key, {"name": r[col["Kernel Name"]], "dev": int(r[col["Device"]])})
        ent[r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
    return list(launches.values())


def family(name):
    m = re.match(r"(?:void )?(?:fssdp::)?([a-z_0-9]+)", name)
    base = m.group(1) if m else name
    if base.startswith("grouped_gemm"):
        return "grouped_gemm" + ("<EPI_F32 (wgrad)>" if ", 3," in name else "")
    return base


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    args = ap.parse_args()
    ls = load(args.csv)
    # the last iteration starts at the last launch of the gate on device 0 (if captured)
    starts = [i for i, x in enumerate(ls) if family(x["name"]).startswith("gate_topk")
              and x["dev"] == 0]
    last = ls[starts[-1]:] if starts else ls
    agg = collections.OrderedDict()
    for x in last:
        k = (family(x["name"]), x["dev"])
        a = agg.setdefault(k, {"launches": 0, "time_us": 0.0, "rx_user": 0.0, "tx_user": 0.0,
                               "rx_raw": 0.0, "tx_raw": 0.0})
        a["launches"] += 1
        a["time_us"] += x.get("gpu__time_duration.sum", 0.0) / 1e3
        a["rx_user"] += x.get("nvlrx__bytes_data_user.sum", 0.0)
        a["tx_user"] += x.get("nvltx__bytes_data_user.sum", 0.0)
        a["rx_raw"] += x.get("nvlrx__bytes.sum", 0.0)
        a["tx_raw"] += x.get("nvltx__bytes.sum", 0.0)
    out = []
    for (fam, dev), a in agg.items():
        t = a["time_us"] * 1e-6
        out.append({"kernel": fam, "device": dev, **{k: round(v, 1) for k, v in a.items()},
                    "rx_user_gbs": round(a["rx_user"] / t / 1e9, 1) if t else None,
                    "tx_user_gbs": round(a["tx_user"] / t / 1e9, 1) if t else None})
    for o in out:
        print(json.dumps(o))


if __name__ == "__main__":
    main()
