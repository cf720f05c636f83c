#!/usr/bin/env python3
"""Summaries of ncu CSV logs for profiles/:
    summarize_ncu.py launches <launches.csv>   per-kernel share of device time
    summarize_ncu.py traffic <traffic.csv>     DRAM bytes per launch
    summarize_ncu.py families <traffic.csv>    DRAM bytes per launch of each kernel family
                                               (the roofline "traffic" bench.py reads)
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


# kernel name prefix -> the stage family bench.py reports
FAMILIES = [("k_os_hist", "radix.hist"), ("k_os_pass", "radix.scatter"), ("k_small_sort", "radix.small"),
            ("k_scan_lookback", "scan"), ("k_fy_targets", "fy.targets"), ("k_fy_scatter", "fy.scatter"),
            ("k_fy_lists", "fy.lists"), ("k_fy_sources", "fy.sources_gather"), ("k_nf_round", "nf.round"),
            ("k_ff_chain", "fit.chain"), ("k_ff_replay", "fit.replay"), ("k_eval", "k_eval")]


def families(path):
    per = defaultdict(dict)
    for r in rows(path):
        per[r["ID"]]["name"] = short(r["Kernel Name"]).replace("void ", "")
        per[r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
        per[r["ID"]]["unit:" + r["Metric Name"]] = r["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for m in per.values():
        fam = next((f for pre, f in FAMILIES if m["name"].startswith(pre)), None)
        if fam is None:
            continue
        a = agg[fam]
        a[0] += 1
        a[1] += m["dram__bytes_read.sum"] * scale[m["unit:dram__bytes_read.sum"]] + \
            m["dram__bytes_write.sum"] * scale[m["unit:dram__bytes_write.sum"]]
        a[2] += m["gpu__time_duration.sum"] * scale[m["unit:gpu__time_duration.sum"]]
    out = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                     f"--clock-control none, one C2 step (tools/profile_round.sh, {path.split('/')[-1]}); "
                     "per kernel family: DRAM bytes per launch"}
    for fam, (n, b, t) in agg.items():
        out[fam] = {"launches": n, "dram_bytes": b, "ms": t / 1e6, "dram_bytes_per_launch": b / n,
                    "dram_gbs": b / max(t, 1e-9)}
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    res = launches(path) if mode == "launches" else families(path) if mode == "families" else traffic(path)
    if mode == "launches" and "--md" in sys.argv:
        print(f"{res['launches']} launches, {res['total_ms']:.2f} ms of kernel time (serialised, cold cache)\n")
        print("| kernel | launches | ms | share |\n|---|---:|---:|---:|")
        for k in res["kernels"][:25]:
            print(f"| `{k['kernel']}` | {k['launches']} | {k['ms']:.3f} | {100 * k['share']:.1f}% |")
    else:
        print(json.dumps(res, indent=1))
