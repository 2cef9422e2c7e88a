"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel shares.
usage: python profiles/launch_shares.py gpurun_out/<tag>_launches.csv"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
mi = hdr.index("Metric Name")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":  # captures may carry dram byte metrics too
        continue
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    name = r[ki].split("(")[0]
    tot[name] += us
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':70s} {'launches':>8s} {'total_ms':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {v / 1e3:10.3f} {v / T * 100:5.1f}%")
print(f"{'TOTAL':70s} {sum(cnt.values()):8d} {T / 1e3:10.3f}")
