"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = None
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Value" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("hs::", "")
    name = name.split("<")[0]
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    v *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}.get(unit, 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'mean us':>9s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:34s} {v[0]:8d} {v[1]:10.3f} {v[1] / v[0] * 1e3:9.1f} {v[1] / tot * 100:6.1f}%")
print(f"{'total':34s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")
