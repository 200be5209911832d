"""Per-kernel share of device time from an ncu --metrics gpu__time_duration.sum CSV launch list.

    python tools/launch_shares.py LAUNCHES.csv [--loop-only]

--loop-only drops the operator/sketch construction kernels (setup, not the iteration loop).
"""
import csv
import sys
from collections import defaultdict

SETUP = ("tomo_", "csr_", "cub::", "sell_fill", "sino_block_cols", "sell_delta", "sell_transpose_cols",
         "sell_slice", "tile_perm", "sparse_sign_gen", "i64_to_u64", "u32_to_i64", "sell_c8_encode", "sell_c2_encode",
         "sell_t8_encode")
loop_only = "--loop-only" in sys.argv
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
    if loop_only and name.startswith(SETUP):
        continue
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
