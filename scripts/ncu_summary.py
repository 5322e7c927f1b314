"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by
kernel name: total device time, share, launches, average.

  python scripts/ncu_summary.py launches.csv [exclude-regex]

Kernels matching exclude-regex (setup: assembly, relayout ...) are left out of
the totals and shares.
"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.DictReader(line for line in open(sys.argv[1]) if not line.startswith("==")))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v *= {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    name = r["Kernel Name"]
    if len(sys.argv) > 2 and re.search(sys.argv[2], name):
        continue
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"launches {sum(cnt.values())}  total device time {T:.1f} us")
for name, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:12.1f} us {100 * v / T:5.1f}%  n={cnt[name]:5d}  avg={v / cnt[name]:8.2f} us  {name[:60]}")
