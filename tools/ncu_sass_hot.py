"""Aggregate ncu SASS-level warp-stall samples of one kernel report:
top instructions and samples by opcode.  Usage: ncu_sass_hot.py report.ncu-rep [N]"""
import csv
import collections
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
idx = {k: i for i, k in enumerate(h)}
rows = [x for x in r[2:] if len(x) == len(h)]
k = "Warp Stall Sampling (All Samples)"
tot = sum(float(x[idx[k]] or 0) for x in rows) or 1.0
byop = collections.Counter()
for x in rows:
    op = x[idx["Source"]].split()[0] if x[idx["Source"]].split() else "?"
    if op.startswith("@"):
        op = x[idx["Source"]].split()[1]
    byop[op.split(".")[0]] += float(x[idx[k]] or 0)
print("samples by opcode (%):")
for op, v in byop.most_common(15):
    print(f"  {op:10s} {100 * v / tot:5.1f}")
print("hottest instructions:")
order = sorted(range(len(rows)), key=lambda i: -float(rows[i][idx[k]] or 0))
for i in order[:top]:
    x = rows[i]
    print(f"  {100 * float(x[idx[k]]) / tot:5.1f}%  #{i:5d} {x[idx['Address']]} {x[idx['Source']].strip()[:90]}")
