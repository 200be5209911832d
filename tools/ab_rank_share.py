"""One rank's share of the config-4 operator on P GPUs, built and timed on one
GPU (HS_FAKE_SHARD="r/P" with forced sharding: the rank's rays for A, every ray
restricted to the rank's image rows for A^T, exactly as build_tomo_sharded
partitions them).  Times the rank's A x and A^T y for SpMV schedule variants.

    python tools/ab_rank_share.py [r/P] [VARIANTS...]

VARIANTS: "N" = HS_D16_PIPE depth N, "auto" = the library's default choice.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import _lib
from paper_2502_02721_b200 import dist as hsd

shard = sys.argv[1] if len(sys.argv) > 1 else "0/8"
variants = sys.argv[2:] or ["auto", "0", "1", "2"]
os.environ["HS_FAKE_SHARD"] = shard
hsd.force_sharding(True)
op = hs.TomographyOperator(2048, 720, 2897, dtype=np.float32)
ctx = _lib.context()
x = np.random.default_rng(0).random(op.cols).astype(np.float32)
y = np.random.default_rng(1).random(op.rows).astype(np.float32)
ref = None
best = {}
for rnd in range(3):
    for d in variants:
        os.environ.pop("HS_D16_PIPE", None)
        if d != "auto":
            os.environ["HS_D16_PIPE"] = d
        ctx.reset_stats(); ctx.set_profiling(True)
        for _ in range(3):
            out = (op.matvec(x, np.float32), op.rmatvec(y, np.float32))
        st = ctx.kernel_stats(); ctx.set_profiling(False)
        if ref is None:
            ref = out
        same = all(np.array_equal(a, b) for a, b in zip(out, ref))
        a_ms = st["spmv_A"]["ms"] / st["spmv_A"]["launches"]
        at_ms = st["spmv_AT"]["ms"] / st["spmv_AT"]["launches"]
        ga = st["spmv_A"]["bytes"] / st["spmv_A"]["launches"] / 1e9
        gt = st["spmv_AT"]["bytes"] / st["spmv_AT"]["launches"] / 1e9
        print(f"round {rnd} {d:>4s}: A {a_ms:.3f} ms ({ga / a_ms:.2f} TB/s of {ga:.2f} GB)  "
              f"AT {at_ms:.3f} ms ({gt / at_ms:.2f} TB/s of {gt:.2f} GB)  bitwise {same}", flush=True)
        if rnd > 0:
            b = best.setdefault(d, [9e9, 9e9])
            b[0], b[1] = min(b[0], a_ms), min(b[1], at_ms)
print(json.dumps({"shard": shard, "best_ms": best}))
hsd.force_sharding(False)
