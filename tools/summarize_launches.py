"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    v = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
    name = r["Kernel Name"].split("(")[0][:90]
    tot[name] += v
    cnt[name] += 1
S = sum(tot.values())
print(f"total {S:.1f} us over {sum(cnt.values())} launches")
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us {100 * v / S:5.1f}%  x{cnt[n]:4d}  {n}")
