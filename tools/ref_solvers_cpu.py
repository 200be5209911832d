"""CPU timings of the UNMODIFIED reference solvers on the same problems as
tools/bench_solvers.py (run in the build container, where /root/reference
exists; it does not travel to the GPU box).  it/s = iterations / sum(wall_ms).

    PYTHONPATH=/root/reference/pkg/src python tools/ref_solvers_cpu.py [--maxiter 100]
"""
import argparse
import json
import os
import time

import numpy as np
from hessketch import problems, solvers
from hessketch.hessenberg import PivotStrategy

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=256)
ap.add_argument("--angles", type=int, default=180)
ap.add_argument("--deblur", type=int, default=256)
ap.add_argument("--maxiter", type=int, default=100)
args = ap.parse_args()
K = args.maxiter
t0 = time.perf_counter()
tomo = problems.make_tomography(args.grid, args.angles, noise_level=0.01, seed=0)
t_build = time.perf_counter() - t0
blur = problems.make_deblur(args.deblur, problems.gaussian_psf(2.0, radius=7), noise_level=0.01, seed=0)
runs = [
    ("slslu", tomo, solvers.slslu, solvers.SolverConfig(maxiter=K)),
    ("slslu sampled(1000)", tomo, solvers.slslu, solvers.SolverConfig(maxiter=K, pivot=PivotStrategy.sampled(1000, seed=1))),
    ("lslu", tomo, solvers.lslu, solvers.SolverConfig(maxiter=K)),
    ("lsqr", tomo, solvers.lsqr, solvers.SolverConfig(maxiter=K)),
    ("scmrh", blur, solvers.scmrh, solvers.SolverConfig(maxiter=K)),
    ("scmrh sampled(1000)", blur, solvers.scmrh, solvers.SolverConfig(maxiter=K, pivot=PivotStrategy.sampled(1000, seed=1))),
    ("cmrh", blur, solvers.cmrh, solvers.SolverConfig(maxiter=K)),
    ("gmres", blur, solvers.gmres, solvers.SolverConfig(maxiter=K)),
]
for name, prob, fn, cfg in runs:
    r = fn(prob.operator, prob.b, cfg, x_true=prob.x_true)
    ms = sum(rec.wall_ms for rec in r.trace.records)
    it = len(r.trace.records)
    print(json.dumps({"solver": name, "impl": "reference (numpy/scipy, CPU)", "cores": os.cpu_count(), "iters": it,
                      "loop_ms": round(ms, 1), "it_per_s": round(it / (ms / 1e3), 2),
                      "tomography_build_s": round(t_build, 1)}), flush=True)
