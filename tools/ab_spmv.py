"""A/B timing of the config-4 SpMVs in one process: alternate environment
settings (e.g. HS_SPMV_CARVEOUT) between rounds and compare kernel times.

    python tools/ab_spmv.py VAR valueA valueB [rounds]

AB_REBUILD=1 builds one operator per value (for build-time variables such as HS_SINO_BLK).
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import _lib

var, va, vb = sys.argv[1], sys.argv[2], sys.argv[3]
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 6
scale = int(os.environ.get("AB_SCALE", "2048"))
f = scale / 2048
def mk():
    return hs.TomographyOperator(scale, round(720 * f), round(2897 * f), dtype=np.float32)

# AB_REBUILD=1: the variable is read at operator build time -> one operator per value
ops = {}
if os.environ.get("AB_REBUILD") == "1":
    for v in (va, vb):
        os.environ[var] = v
        ops[v] = mk()
else:
    ops[va] = ops[vb] = mk()
op = ops[va]
ctx = _lib.context()
x = np.random.default_rng(0).random(op.cols).astype(np.float32)
y = np.random.default_rng(1).random(op.rows).astype(np.float32)
res = {va: {"A": [], "AT": []}, vb: {"A": [], "AT": []}}
outs = {}
for r in range(rounds):
    for v in (va, vb) if r % 2 == 0 else (vb, va):
        os.environ[var] = v
        op = ops[v]
        ctx.reset_stats(); ctx.set_profiling(True)
        for _ in range(3):
            outs[v] = (op.matvec(x, np.float32), op.rmatvec(y, np.float32))
        st = ctx.kernel_stats(); ctx.set_profiling(False)
        res[v]["A"].append(st["spmv_A"]["ms"] / st["spmv_A"]["launches"])
        res[v]["AT"].append(st["spmv_AT"]["ms"] / st["spmv_AT"]["launches"])
print("bitwise equal:", all(np.array_equal(a, b) for a, b in zip(outs[va], outs[vb])))
for v in (va, vb):
    print(f"{var}={v}: A {np.median(res[v]['A']):.3f} ms  AT {np.median(res[v]['AT']):.3f} ms")
