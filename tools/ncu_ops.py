"""Executed instructions and stall samples per SASS opcode (and the hottest
instructions) of the K-th kernel in an .ncu-rep (ncu --page source sass)."""
import collections
import csv
import subprocess
import sys

rep, k = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows, n = [], 0
for x in csv.reader(out.splitlines()):
    if x and x[0] == "Kernel Name":
        n += 1
        continue
    if n == k and len(x) > 6 and x[0].startswith("0x"):
        rows.append(x)
tot = sum(int(x[5]) for x in rows)
print("instructions executed", tot, "sass lines", len(rows))
op, st = collections.Counter(), collections.Counter()
for x in rows:
    w = x[1].split()
    o = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
    op[o] += int(x[5])
    st[o] += int(x[2])
for o, c in op.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"{o:12s} {c:10d} {100 * c / tot:5.1f}%  stall-samples {st[o]}")
print("hottest stalls:")
for x in sorted(rows, key=lambda x: -int(x[2]))[:25]:
    print(x[0][-5:], x[2].rjust(6), x[5].rjust(9), x[1])
