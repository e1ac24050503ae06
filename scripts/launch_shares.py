"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
totals and shares of the step.  Usage: python scripts/launch_shares.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

tot = defaultdict(float)
cnt = defaultdict(int)
with open(sys.argv[1]) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = row["Kernel Name"]
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"fcg::(<unnamed>|\(anonymous namespace\))::", "", name)
    name = name.replace("void ", "")
    ns = float(row["Metric Value"])
    tot[name] += ns
    cnt[name] += 1
T = sum(tot.values())
print(f"total {T / 1e6:.3f} ms over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v / T:7.3f}  {v / 1e6:9.3f} ms  {cnt[k]:5d}x  {k[:110]}")
