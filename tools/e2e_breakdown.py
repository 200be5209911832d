"""Time the phases of one public solver call (setup vs loop).

    python tools/e2e_breakdown.py [CFG] [SCALE]
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import _lib
from paper_2502_02721_b200.problems import make_workload

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
scale = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = make_workload(cid, scale=scale)
solve = hs.slslu if w.solver == "slslu" else hs.scmrh
for i in range(3):
    t0 = time.perf_counter()
    res = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    t1 = time.perf_counter()
    print(f"solve {i}: wall {t1-t0:.3f}s loop {res.loop_ms/1e3:.3f}s overhead {t1-t0-res.loop_ms/1e3:.3f}s")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
res = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
