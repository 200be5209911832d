"""Time the config-4 SpMVs back to back while sampling the SM clock (is the
in-solve slowdown of the SpMV kernels the power-capped clock?).

    python tools/spmv_clocks.py [reps]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import _lib
from bench import ClockSampler

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
op = hs.TomographyOperator(2048, 720, 2897, dtype=np.float32)
ctx = _lib.context()
x = np.random.default_rng(0).random(op.cols).astype(np.float32)
y = np.random.default_rng(1).random(op.rows).astype(np.float32)
for _ in range(3):
    op.matvec(x, np.float32); op.rmatvec(y, np.float32)
ctx.reset_stats(); ctx.set_profiling(True)
with ClockSampler(0) as clk:
    t0 = time.perf_counter()
    for _ in range(reps):
        op.matvec(x, np.float32); op.rmatvec(y, np.float32)
    wall = time.perf_counter() - t0
st = ctx.kernel_stats(); ctx.set_profiling(False)
print("A %.3f ms  AT %.3f ms  wall %.2f s (GPU busy %.0f%%)  clocks %s" % (
    st["spmv_A"]["ms"] / st["spmv_A"]["launches"], st["spmv_AT"]["ms"] / st["spmv_AT"]["launches"], wall,
    100 * (st["spmv_A"]["ms"] + st["spmv_AT"]["ms"]) / 1e3 / wall, clk.summary()))
