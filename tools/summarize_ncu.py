"""Summarise an ncu --csv launch list (gpu__time_duration.sum, dram__bytes_*)
into the per-kernel JSON that bench.py reads for roofline.traffic.

    python tools/summarize_ncu.py launches.csv out.json --grid 256 --label "..."
"""

import argparse
import csv
import io
import json
import re
from collections import defaultdict


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").strip()
    base = re.sub(r"\s+", "", base)
    return base[4:] if base.startswith("cf::") else base


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out")
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--label", default="")
    ap.add_argument("--round", type=int, default=1)
    a = ap.parse_args()
    text = open(a.csv).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: defaultdict(dict))
    to_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    to_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v *= to_us.get(u, 1.0) if r["Metric Name"].startswith("gpu__time") else to_b.get(u, 1.0)
        per[r["ID"]][r["Metric Name"]] = v
        per[r["ID"]]["name"] = short(r["Kernel Name"])
    agg = defaultdict(lambda: {"launches": 0, "us": 0.0, "bytes": 0.0})
    for launch in per.values():
        k = agg[launch["name"]]
        k["launches"] += 1
        k["us"] += launch.get("gpu__time_duration.sum", 0.0)
        k["bytes"] += launch.get("dram__bytes_read.sum", 0.0) + launch.get("dram__bytes_write.sum", 0.0)
    total = sum(k["us"] for k in agg.values())
    kernels = {}
    for name, k in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        kernels[name] = {"launches": k["launches"], "share_pct": round(100 * k["us"] / total, 2),
                         "avg_us": round(k["us"] / k["launches"], 2),
                         "dram_mb_per_launch": round(k["bytes"] / k["launches"] / 1e6, 1)}
    spass = {n: k for n, k in agg.items() if n.startswith("cg_spass")}
    if spass:  # the single-pass form: one launch per iteration
        cg, form, design = spass, "single-pass", 40
        dirs = sum(k["launches"] for k in spass.values())
    else:
        cg = {n: k for n, k in agg.items() if n.startswith(("cg_dir", "cg_update"))}
        form, design = "two-kernel", 60
        dirs = sum(k["launches"] for n, k in cg.items() if n.startswith("cg_dir"))
    cg_bytes = sum(k["bytes"] for k in cg.values())
    n3 = a.grid ** 3
    out = {"round": a.round, "source": a.label, "grid": f"{a.grid}^3", "form": form, "kernels": kernels,
           "cg_iterations_profiled": dirs,
           "dram_bytes_per_iteration": cg_bytes / dirs if dirs else None,
           "cg_us_per_iteration_cold": sum(k["us"] for k in cg.values()) / dirs if dirs else None,
           "algorithmic_bytes_per_iteration_88N": 88 * n3,
           f"design_bytes_per_iteration_{design}N": design * n3}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "kernels"}))
    for n, k in list(kernels.items())[:8]:
        print(n, k)


if __name__ == "__main__":
    main()
