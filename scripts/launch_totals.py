"""Aggregate an ncu --metrics gpu__time_duration.sum CSV log by kernel name."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; idx = {k: i for i, k in enumerate(h)}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[idx["Metric Value"]].replace(",", ""))
    u = r[idx["Metric Unit"]]
    us = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}[u]
    n = r[idx["Kernel Name"]][:70]
    tot[n] += us; cnt[n] += 1
T = sum(tot.values())
for n, us in sorted(tot.items(), key=lambda x: -x[1])[:20]:
    print(f"{us/1e3:10.2f} ms {100*us/T:5.1f}%  x{cnt[n]:6d}  {us/cnt[n]:9.1f} us/launch  {n}")
print(f"total {T/1e3:.1f} ms over {sum(cnt.values())} launches")
