"""Config 4 (or a scaled copy) solved by P in-process ranks on ONE GPU
(hs_comm_init_local: P contexts, one host thread per rank, the NCCL path's
partition and message sequence with device copies for the collectives),
checked bit for bit against the single-GPU solve: pivots t / g, H, W, y, x,
sres.  The emulated run's time is not a scaling measurement (all ranks share
one GPU); it shows the full-size sharded loop runs and is P-independent.

    python tools/run_local_ranks.py [--ranks 8] [--scale 2048] [--maxiter 300]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import dist as hsd
from paper_2502_02721_b200.problems import make_workload

ap = argparse.ArgumentParser()
ap.add_argument("--ranks", type=int, default=8)
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--maxiter", type=int, default=300)
args = ap.parse_args()

t0 = time.perf_counter()
w = make_workload(4, scale=args.scale, maxiter=args.maxiter)
r1 = hs.slslu(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
single = dict(t=r1.factorization.t[: args.maxiter + 1].copy(), g=r1.factorization.g[: args.maxiter + 1].copy(),
              H=r1.factorization.H_matrix().copy(), W=r1.factorization.W_matrix().copy(), y=r1.factorization._res.y,
              x=r1.x.copy(), sres=r1.trace.column("sres_norm"), loop_ms=r1.loop_ms)
grid, angles, bins = w.meta["grid"], w.meta["angles"], w.meta["bins"]
S, b, x_true, cfg = w.sketch, w.b, w.x_true, w.cfg
del r1, w  # free the single-GPU operator before the shards are built
import gc

gc.collect()
t_single = time.perf_counter() - t0


def rank(r, ctx):
    op = hs.TomographyOperator(grid, angles, bins, dtype=np.float32)
    t = time.perf_counter()
    res = hs.slslu(op, b, cfg, x_true=x_true, sketch=S)
    f = res.factorization
    return dict(t=f.t[: args.maxiter + 1].copy(), g=f.g[: args.maxiter + 1].copy(), H=f.H_matrix().copy(),
                W=f.W_matrix().copy(), y=f._res.y, x=res.x.copy(), sres=res.trace.column("sres_norm"),
                loop_ms=res.loop_ms, wall_s=time.perf_counter() - t, shard=hsd.shard_plan(grid, angles, bins,
                                                                                       args.ranks, r).__dict__)


ctxs = hsd.local_group(args.ranks)
t1 = time.perf_counter()
outs = hsd.run_ranks(rank, ctxs)
t_ranks = time.perf_counter() - t1
for c in ctxs:
    c.close()
same = {}
for key in ("t", "g", "H", "W", "y", "x", "sres"):
    same[key] = all(np.array_equal(np.asarray(o[key]), np.asarray(single[key])) for o in outs)
print(json.dumps({
    "config": f"cfg4 grid={grid} angles={angles} bins={bins} maxiter={args.maxiter}",
    "ranks": args.ranks, "bitwise_equal_to_single_gpu": same, "all_equal": all(same.values()),
    "single_gpu_loop_ms": round(single["loop_ms"], 2),
    "emulated_rank_loop_ms": [round(o["loop_ms"], 2) for o in outs],
    "note": "emulated ranks share one GPU: their loop time is NOT a multi-GPU measurement",
    "shards": [o["shard"] for o in outs], "setup_and_single_s": round(t_single, 1), "ranks_s": round(t_ranks, 1),
}))
