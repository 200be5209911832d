"""Host launch time vs device loop time of one solve (HS_TIMING=1 prints the
host-side phases of hs_solve): is a latency-bound config limited by the host
issuing launches or by the device?

    python tools/host_vs_device.py [config ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HS_TIMING"] = "1"
import paper_2502_02721_b200 as hs
from paper_2502_02721_b200.problems import make_workload

for cid in [int(a) for a in sys.argv[1:]] or [1, 2, 3]:
    w = make_workload(cid)
    solve = hs.slslu if w.solver == "slslu" else hs.scmrh
    for rep in range(3):
        r = solve(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
        print(f"cfg{cid} rep{rep}: device loop {r.loop_ms:.2f} ms", file=sys.stderr, flush=True)
