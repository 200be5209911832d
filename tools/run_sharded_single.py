"""A config (5, 2: sCMRH on the PSF operator; 3, 4: sLSLU on tomography) through the
row-sharded loop forced on one rank, beside the single-GPU loop (same problem):
it/s of both and bitwise agreement of the pivots.

    python tools/run_sharded_single.py [CFG]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import dist as hsd
from paper_2502_02721_b200.problems import make_workload

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = {"config": cid}
res = {}
for tag, forced in (("single", False), ("sharded_p1", True)):
    hsd.force_sharding(forced)
    w = make_workload(cid)
    solve = hs.slslu if w.solver == "slslu" else hs.scmrh
    r = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)  # warm
    r = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    res[tag] = r
    out[tag + "_it_per_s"] = round(len(r.trace.records) / (r.loop_ms / 1e3), 1)
    del w
hsd.force_sharding(False)
a, b = res["single"], res["sharded_p1"]
out["pivots_equal"] = bool(np.array_equal(a.factorization._res.pivots_t, b.factorization._res.pivots_t))
out["x_equal"] = bool(np.array_equal(a.x, b.x))
print(json.dumps(out))
