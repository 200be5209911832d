import os, sys, json, dataclasses
sys.path.insert(0, os.getcwd())
import paper_2502_02721_b200 as hs
from paper_2502_02721_b200.problems import make_workload
w = make_workload(2)
out = {}
for tag, cfg, xt in (("default", w.cfg, w.x_true), ("no_relerr", dataclasses.replace(w.cfg, record_rel_err=False), w.x_true), ("no_xtrue", w.cfg, None)):
    r = hs.scmrh(w.operator, w.b, cfg, x_true=xt, sketch=w.sketch)
    r = hs.scmrh(w.operator, w.b, cfg, x_true=xt, sketch=w.sketch)
    out[tag] = round(len(r.trace.records) / (r.loop_ms / 1e3), 1)
print(os.environ.get("HS_SKETCH_BATCH", "8"), json.dumps(out))
