"""One solve of a BASELINE config with a reduced iteration count (for ncu
launch lists / per-kernel captures).

    python tools/profile_workload.py CFG [MAXITER]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200.problems import make_workload

cid = int(sys.argv[1])
maxiter = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = make_workload(cid, maxiter=maxiter)
solve = hs.slslu if w.solver == "slslu" else hs.scmrh
r = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
print(f"cfg{cid}: {len(r.trace.records)} iterations, {r.loop_ms:.2f} ms loop")
