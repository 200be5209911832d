"""Device timings of every solver family on the reference's own problem
builders (sampled pivoting, unsketched CMRH/LSLU,
GMRES/LSQR), one JSON line each.  CUDA-event loop time (``loop_ms``) after one
warm-up solve; fp64 (the reference's arithmetic).

    python tools/bench_solvers.py [--grid 256] [--angles 180] [--maxiter 100]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs
from paper_2502_02721_b200 import problems

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--angles", type=int, default=180)
ap.add_argument("--deblur", type=int, default=256)
ap.add_argument("--maxiter", type=int, default=100)
args = ap.parse_args()
K = args.maxiter

tomo = problems.make_tomography(args.grid, args.angles, noise_level=0.01, seed=0)
blur = problems.make_deblur(args.deblur, problems.gaussian_psf(2.0, radius=7), noise_level=0.01, seed=0)
ell = 10 * (K + 1)
runs = [
    ("slslu", "tomography", lambda: hs.slslu(tomo.operator, tomo.b, hs.SolverConfig(maxiter=K, sketch_kind="gaussian"),
                                             x_true=tomo.x_true)),
    ("slslu sampled(1000)", "tomography",
     lambda: hs.slslu(tomo.operator, tomo.b, hs.SolverConfig(maxiter=K, sketch_kind="gaussian",
                                                             pivot=hs.PivotStrategy.sampled(1000, seed=1)),
                      x_true=tomo.x_true)),
    ("lslu", "tomography", lambda: hs.lslu(tomo.operator, tomo.b, hs.SolverConfig(maxiter=K), x_true=tomo.x_true)),
    ("lsqr", "tomography", lambda: hs.lsqr(tomo.operator, tomo.b, hs.SolverConfig(maxiter=K), x_true=tomo.x_true)),
    ("scmrh", "deblur", lambda: hs.scmrh(blur.operator, blur.b, hs.SolverConfig(maxiter=K, sketch_kind="gaussian"),
                                         x_true=blur.x_true)),
    ("scmrh sampled(1000)", "deblur",
     lambda: hs.scmrh(blur.operator, blur.b, hs.SolverConfig(maxiter=K, sketch_kind="gaussian",
                                                             pivot=hs.PivotStrategy.sampled(1000, seed=1)),
                      x_true=blur.x_true)),
    ("cmrh", "deblur", lambda: hs.cmrh(blur.operator, blur.b, hs.SolverConfig(maxiter=K), x_true=blur.x_true)),
    ("gmres", "deblur", lambda: hs.gmres(blur.operator, blur.b, hs.SolverConfig(maxiter=K), x_true=blur.x_true)),
]
for name, prob, fn in runs:
    fn()  # warm-up
    t0 = time.perf_counter()
    r = fn()
    wall = time.perf_counter() - t0
    it = len(r.trace.records)
    rel = r.trace.column("rel_err")
    size = (f"{args.grid}^2 x {args.angles} angles" if prob == "tomography" else f"{args.deblur}^2, 15x15 psf")
    print(json.dumps({
        "solver": name, "problem": f"{prob} {size}", "dtype": "f64", "iters": it, "termination": r.termination,
        "loop_ms": round(r.loop_ms, 2), "it_per_s": round(it / (r.loop_ms / 1e3), 1),
        "e2e_it_per_s": round(it / wall, 1), "dots_final": r.trace.final().dots,
        "rel_err_min_last": [round(min(rel), 5), round(rel[-1], 5)],
    }), flush=True)
