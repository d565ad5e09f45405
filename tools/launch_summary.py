"""Per-kernel totals and shares of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = defaultdict(float)
cnt = defaultdict(int)
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mdg::<unnamed>::", "")
        tot[name] += float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "ns"), 1e-3)
        cnt[name] += 1
all_us = sum(tot.values())
print(f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'share':>7s}")
for k in sorted(tot, key=lambda x: -tot[x]):
    print(f"{k:40s} {cnt[k]:8d} {tot[k]:10.1f} {100 * tot[k] / all_us:6.1f}%")
print(f"{'all':40s} {sum(cnt.values()):8d} {all_us:10.1f}")
