"""Aggregate an `ncu --csv --metrics ...` launch list per kernel (development tool).
Usage: python tools/ncu_agg.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    agg.setdefault((d["ID"], d["Kernel Name"][:48]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
tot = collections.OrderedDict()
for (_, k), m in agg.items():
    t = tot.setdefault(k, [0, 0.0, 0.0, 0.0])
    t[0] += 1
    t[1] += m.get("gpu__time_duration.sum", 0)
    t[2] += m.get("dram__bytes_read.sum", 0)
    t[3] += m.get("dram__bytes_write.sum", 0)
for k, t in tot.items():
    print(f"{k:50s} n={t[0]:4d} us/launch={t[1] / t[0] / 1e3:9.1f} rdGB={t[2] / t[0] / 1e9:6.2f} wrGB={t[3] / t[0] / 1e9:6.2f}")
