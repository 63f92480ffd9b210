"""Aggregate an ncu launch list (`--metrics gpu__time_duration.sum --csv`)
per kernel: launches, mean duration and share of the listed time."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
acc = collections.OrderedDict()
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").replace("nwb::", "")
    us = float(r[14]) * (1e-3 if r[13] == "ns" else 1.0)
    e = acc.setdefault(name, [0, 0.0])
    e[0] += 1
    e[1] += us
tot = sum(v[1] for v in acc.values())
print(f"{'kernel':36s} {'launches':>8s} {'mean_us':>9s} {'share_of_listed':>16s}")
for k, (n, us) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:36s} {n:8d} {us / n:9.1f} {us / tot:16.3f}")
