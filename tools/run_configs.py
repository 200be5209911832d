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
    # the same solve without the per-kernel event brackets
    t2 = time.perf_counter()
    rn = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    wall_np = time.perf_counter() - t2
    loop_np = rn.loop_ms
    del rn
    rel = r.trace.column("rel_err")
    out = {
        "config": cid, "desc": CONFIGS[cid], "iters": len(r.trace.records), "termination": r.termination,
        "loop_ms": round(r.loop_ms, 2), "it_per_s": round(len(r.trace.records) / (r.loop_ms / 1e3), 1),
        "e2e_it_per_s": round(len(r.trace.records) / wall, 1), "setup_s": round(setup, 2),
        "it_per_s_noprof": round(len(r.trace.records) / (loop_np / 1e3), 1),
        "e2e_it_per_s_noprof": round(len(r.trace.records) / wall_np, 1),
        "rel_err_first_min_last": [round(rel[0], 5), round(min(rel), 5), round(rel[-1], 5)],
        "sres_last": r.trace.final().sres_norm, "rank_fallback": any(r.trace.column("rank_fallback")),
        "kernels_ms": {k: round(v["ms"], 2) for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])},
    }
    if cid == 5:
        # BASELINE config 5: "compared against an fp32-storage run" -- same problem,
        # basis stored in fp32 instead of bf16
        import dataclasses
        r32 = solve(w.operator, w.b, dataclasses.replace(w.cfg, basis_dtype="float32"), x_true=w.x_true,
                    sketch=w.sketch)
        t16, t32 = r.factorization.t, r32.factorization.t
        nt = min(len(t16), len(t32))
        diff = np.nonzero(t16[:nt] != t32[:nt])[0]
        rel32 = r32.trace.column("rel_err")
        out["fp32_storage"] = {
            "it_per_s": round(len(r32.trace.records) / (r32.loop_ms / 1e3), 1),
            "rel_err_first_min_last": [round(rel32[0], 5), round(min(rel32), 5), round(rel32[-1], 5)],
            "rel_err_min_bf16_over_fp32": round(min(rel) / min(rel32), 4),
            "first_pivot_divergence_k": int(diff[0]) + 1 if len(diff) else None,
        }
        kmin = int(np.argmin(rel32))
        out["fp32_storage"]["argmin_rel_err_k"] = [int(np.argmin(rel)) + 1, kmin + 1]
        del r32
    print(json.dumps(out), flush=True)
    del r, w
