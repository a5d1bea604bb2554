"""Per-kernel table from an ncu launch list (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum) of tools/ncu_table.py at 256^3:
average time, DRAM bytes vs the kernel's algorithmic bytes,
achieved GB/s on algorithmic and on DRAM bytes, fraction of the measured peak.

    python tools/kernel_table.py table.csv profiles/r02_kernel_table.json [--n 256] [--label ...]
"""
import argparse
import csv
import io
import json
import os
import re
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def alg_bytes(name, n):
    """Algorithmic bytes of one launch at n^3 (None: not a streaming kernel of the path)."""
    N = n ** 3
    F = (n + 1) * n * n
    U = 3 * N - 3 * n * n          # stored upper entries of the symmetric form
    nnz = 7 * N - 6 * n * n
    table = [
        (r"cg_spass_kernel<\d+,\d+,\d+,0", 32 * N, "r_k, p_{k-1} read; r_{k+1}, p_k written"),
        (r"cg_spass_kernel<\d+,\d+,\d+,1", 48 * N, "+ x read and written (every 2nd pass)"),
        (r"cg_dir_lean2", 24 * N, "r, p_old read; p written"),
        (r"cg_update_tma<\d+,\d+,1", 24 * N, "p, r read; r written"),
        (r"cg_update_tma<\d+,\d+,2", 48 * N, "p, r, x, p_prev read; r, x written"),
        (r"cg_pass_init", 24 * N, "b read; r, x written (+ A z_0 from b)"),
        (r"cg_init_flat", 32 * N, "b read; r, x, (z) written"),
        (r"cg_x_fixup", 24 * N, "x, p read; x written (only after an odd count)"),
        (r"advect_kernel", 48 * F, "3 components read (gathers) and written"),
        (r"advect_tma_kernel", 48 * F, "3 components read (TMA boxes) and written"),
        (r"diffuse_(kernel|march)", 48 * F, "3 components read and written"),
        (r"divergence_(kernel|march)", 24 * F + 8 * N, "3 components read; b written"),
        (r"correct_(kernel|march)", 48 * F + 8 * N, "3 components + p read; 3 components written"),
        (r"stencil_apply_pair", 16 * N, "x read; y written"),
        (r"csr_spmv_kernel", 12 * nnz + 4 * (N + 1) + 16 * N, "int32 CSR + x read; y written"),
        (r"sym_spmv_kernel", 24 * N + 24 * U + 8 * (N + 1), "diag, upper + transpose arrays, x read; y written"),
        (r"dic_wave_(fwd|bwd)", 24 * N, "r (w), d read; w (z) written"),
        (r"dic_skew_fwd", 32 * N, "r, (d, 1/d) read; w written"),
        (r"dic_skew_bwd", 32 * N, "w, (d, 1/d) read; z written"),
    ]
    for pat, b, what in table:
        if re.search(pat, name):
            return b, what
    return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out")
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--label", default="")
    a = ap.parse_args()
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = 6541.1
    rows = []
    paths = a.csv.split(",")
    for part, path in enumerate(paths):  # several launch lists: IDs kept apart
        text = open(path).read()
        for r in csv.DictReader(io.StringIO(text[text.index('"ID"'):])):
            # with a separate CG list (the last one, dense right-hand side), the
            # step list's CG launches (the cavity's first, mostly-zero solves) are dropped
            if len(paths) > 1 and part < len(paths) - 1 and "cg_" in r["Kernel Name"]:
                continue
            r["ID"] = f"{part}:{r['ID']}"
            rows.append(r)
    per = defaultdict(dict)
    to_us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    to_b = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v *= to_us.get(u, 1.0) if r["Metric Name"].startswith("gpu__time") else to_b.get(u, 1.0)
        per[r["ID"]][r["Metric Name"]] = v
        base = r["Kernel Name"].split("(")[0].replace("void ", "").replace("cf::", "").replace(" ", "")
        per[r["ID"]]["name"] = base
    # launches that exit at once (the solve had already stopped: every graph-body
    # kernel checks the done flag) would dilute the averages: dropped
    longest = defaultdict(float)
    for l in per.values():
        longest[l["name"]] = max(longest[l["name"]], l.get("gpu__time_duration.sum", 0.0))
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for l in per.values():
        if l.get("gpu__time_duration.sum", 0.0) < 0.05 * longest[l["name"]]:
            continue
        k = agg[l["name"]]
        k[0] += 1
        k[1] += l.get("gpu__time_duration.sum", 0.0)
        k[2] += l.get("dram__bytes_read.sum", 0.0) + l.get("dram__bytes_write.sum", 0.0)
    out = []
    for name, (cnt, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        ab, what = alg_bytes(name, a.n)
        t = us / cnt
        row = {"kernel": name, "launches": cnt, "avg_us": round(t, 2), "dram_mb": round(by / cnt / 1e6, 1)}
        if ab:
            row.update({"alg_mb": round(ab / 1e6, 1), "dram_over_alg": round(by / cnt / ab, 3),
                        "alg_gbs": round(ab / t / 1e3, 1), "dram_gbs": round(by / cnt / t / 1e3, 1),
                        "frac_alg": round(ab / t / 1e3 / peak, 3), "frac_dram": round(by / cnt / t / 1e3 / peak, 3),
                        "bytes": what})
        out.append(row)
    doc = {"source": a.label, "grid": f"{a.n}^3", "peak_gbs": peak, "peak_kind": "MEASURED_PEAKS.json hbm_gbs",
           "note": "ncu launch list: serialised, cold-cache per launch (--clock-control none)", "kernels": out}
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    md = os.path.splitext(a.out)[0] + ".md"
    with open(md, "w") as f:
        f.write(f"# Per-kernel table, {a.n}^3 ({a.label})\n\nPeak {peak} GB/s (MEASURED_PEAKS.json). ")
        f.write("Cold-cache ncu launch list; frac = GB/s / peak.\n\n")
        f.write("| Kernel | launches | avg us | DRAM MB | alg MB | DRAM/alg | alg GB/s | frac (alg) | frac (DRAM) |\n")
        f.write("| --- | --- | --- | --- | --- | --- | --- | --- | --- |\n")
        for r in out:
            if "alg_mb" not in r:
                continue
            f.write(f"| `{r['kernel'][:60]}` | {r['launches']} | {r['avg_us']} | {r['dram_mb']} | {r['alg_mb']} | "
                    f"{r['dram_over_alg']} | {r['alg_gbs']} | {r['frac_alg']} | {r['frac_dram']} |\n")
    print(json.dumps([r["kernel"] for r in out[:12]]))


if __name__ == "__main__":
    main()
