"""Hottest SASS instructions of the K-th kernel in an .ncu-rep with their
stall reasons and shared-memory wavefronts (ncu --page source sass).

    python tools/ncu_hot.py rep.ncu-rep [K] [N] [lo_addr hi_addr]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows, n, hdr = [], 0, None
for x in csv.reader(out.splitlines()):
    if x and x[0] == "Kernel Name":
        n += 1
        continue
    if x and x[0] == "Address":
        hdr = x
        continue
    if n == k and len(x) > 6 and x[0].startswith("0x"):
        rows.append(x)
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(x[ix["Warp Stall Sampling (All Samples)"]]) for x in rows)
wf = sum(int(x[ix["L1 Wavefronts Shared"]] or 0) for x in rows)
wfi = sum(int(x[ix["L1 Wavefronts Shared Ideal"]] or 0) for x in rows)
print(f"samples {tot}  smem wavefronts {wf} (ideal {wfi})")
agg = {s: sum(int(x[ix[s]] or 0) for x in rows) for s in stalls}
print("stalls:", ", ".join(f"{s[6:]}={v}" for s, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
for x in sorted(rows, key=lambda x: -int(x[ix["Warp Stall Sampling (All Samples)"]]))[:top]:
    st = sorted(((int(x[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(x[0][-5:], x[ix["Warp Stall Sampling (All Samples)"]].rjust(5), x[ix["Instructions Executed"]].rjust(8),
          (x[ix["L1 Wavefronts Shared"]] or "").rjust(7), " ".join(f"{b}={a}" for a, b in st if a), "|", x[1])
