#!/usr/bin/env python3
"""Summaries of ncu CSV logs for profiles/:
    summarize_ncu.py launches <launches.csv>   per-kernel share of device time
    summarize_ncu.py traffic <traffic.csv>     DRAM bytes per launch
Kernel names are shortened to the function name (template args dropped)."""
import csv
import json
import re
import sys
from collections import defaultdict


def rows(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    return list(csv.DictReader(lines))


def short(name):
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("unnamed>::", "").replace("hbp_b200::", "")
    name = re.sub(r"<.*>", "<…>", name)
    return name.split("::")[-1] if "lambda" not in name else name


def launches(path):
    by_id = {}
    for r in rows(path):
        if r["Metric Name"] == "gpu__time_duration.sum":
            by_id[r["ID"]] = (short(r["Kernel Name"]), float(r["Metric Value"]), r["Grid Size"], r["Block Size"])
    agg = defaultdict(lambda: [0, 0.0])
    for k, t, _, _ in by_id.values():
        agg[k][0] += 1
        agg[k][1] += t
    total = sum(v[1] for v in agg.values())
    out = {"launches": len(by_id), "total_ms": total / 1e6, "kernels": []}
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out["kernels"].append({"kernel": k, "launches": n, "ms": t / 1e6, "share": t / total})
    return out


def traffic(path):
    per = defaultdict(dict)
    for r in rows(path):
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        per[r["ID"]]["unit:" + r["Metric Name"]] = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
    tot_b = tot_t = 0.0
    for m in per.values():
        rd = m["dram__bytes_read.sum"] * scale[m["unit:dram__bytes_read.sum"]]
        wr = m["dram__bytes_write.sum"] * scale[m["unit:dram__bytes_write.sum"]]
        tot_b += rd + wr
        tot_t += m["gpu__time_duration.sum"] * scale[m["unit:gpu__time_duration.sum"]]
    n = len(per)
    return {"launches": n, "dram_bytes_total": tot_b, "dram_bytes_per_launch": tot_b / max(n, 1),
            "ms_total": tot_t / 1e6, "dram_gbs": tot_b / max(tot_t, 1e-9)}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    res = launches(path) if mode == "launches" else traffic(path)
    if mode == "launches" and "--md" in sys.argv:
        print(f"{res['launches']} launches, {res['total_ms']:.2f} ms of kernel time (serialised, cold cache)\n")
        print("| kernel | launches | ms | share |\n|---|---:|---:|---:|")
        for k in res["kernels"][:25]:
            print(f"| `{k['kernel']}` | {k['launches']} | {k['ms']:.3f} | {100 * k['share']:.1f}% |")
    else:
        print(json.dumps(res, indent=1))
