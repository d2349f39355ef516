"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch list:
per-kernel share of the GPU time (cold-cache, serialised launches: compare shares,
not absolute times).  usage: python tools/launch_summary.py launches.csv "<command>" > out.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot = collections.Counter()
cnt = collections.Counter()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
    name = r[ix["Kernel Name"]]
    tot[name] += us
    cnt[name] += 1
s = sum(tot.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none: {sys.argv[2] if len(sys.argv) > 2 else ''}")
print("(cold-cache, serialised launches; compare shares)")
for name, us in tot.most_common():
    print(f"{100 * us / s:6.2f}% {us:13.1f} us {cnt[name]:6d} launches  {name[:60]}")
