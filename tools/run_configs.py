"""Run BASELINE's five configs at full size on the device; print it/s and trace summaries.

    python tools/run_configs.py [1 2 3 4 5]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import _lib
from paper_2502_02721_b200.problems import CONFIGS, make_workload

ids = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
ctx = _lib.context(0)
for cid in ids:
    t0 = time.perf_counter()
    w = make_workload(cid)
    setup = time.perf_counter() - t0
    solve = hs.slslu if w.solver == "slslu" else hs.scmrh
    ctx.reset_stats()
    ctx.set_profiling(True)
    r = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)  # warm
    ctx.reset_stats()
    t1 = time.perf_counter()
    r = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    wall = time.perf_counter() - t1
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    rel = r.trace.column("rel_err")
    out = {
        "config": cid, "desc": CONFIGS[cid], "iters": len(r.trace.records), "termination": r.termination,
        "loop_ms": round(r.loop_ms, 2), "it_per_s": round(len(r.trace.records) / (r.loop_ms / 1e3), 1),
        "e2e_it_per_s": round(len(r.trace.records) / wall, 1), "setup_s": round(setup, 2),
        "rel_err_first_min_last": [round(rel[0], 5), round(min(rel), 5), round(rel[-1], 5)],
        "sres_last": r.trace.final().sres_norm, "rank_fallback": any(r.trace.column("rank_fallback")),
        "kernels_ms": {k: round(v["ms"], 2) for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])},
    }
    print(json.dumps(out), flush=True)
    del r, w
