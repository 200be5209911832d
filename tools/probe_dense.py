"""Time the dense GEMV (order-faithful fp64) at several shapes to split the
per-row add chain (grows with cols) from the product phase (grows with rows).

    python tools/probe_dense.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import _lib

ctx = _lib.context()
rng = np.random.default_rng(0)
for rows, cols in [(1024, 1024), (1024, 256), (1024, 2048), (128, 1024), (4096, 1024)]:
    M = rng.standard_normal((rows, cols))
    op = hs.DenseOperator(M)
    x = rng.standard_normal(cols)
    y0 = op.matvec(x, np.float64)
    ctx.reset_stats()
    ctx.set_profiling(True)
    for _ in range(50):
        y = op.matvec(x, np.float64)
    st = ctx.kernel_stats()
    ctx.set_profiling(False)
    g = st["dense_gemv"]
    print(f"{rows}x{cols}: {1e3 * g['ms'] / g['launches']:.1f} us per apply", np.array_equal(y, y0))
