"""Seconds per sLSLU iteration of the UNMODIFIED Python reference at a reduced
size of config 4, beside the C port (oracle/coracle.c) on the same operator,
sketch and host -- the measured anchor for the reference arm's C port
(bench.py --impl reference).  Run in the build container, where
/root/reference exists (it does not travel to the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tools/ref_python_scaled.py [--grid 512]

The operator is the exact-chord CSR of the config's geometry scaled to
`grid` (built by the C restatement of the reference ray tracer, bit-identical
to problems.tomography_matrix), injected into the reference through
LinearOperator.from_matrix; S2 is a sparse-sign matrix injected through
`sketch=` (both as the reference's public API allows).  Writes
profiles/r2/reference_python_scaled.json.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import scipy.sparse
from hessketch import linops, sketch, solvers

from oracle import cpu_baseline as cb

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=512)
ap.add_argument("--maxiter", type=int, default=12)
ap.add_argument("--ell", type=int, default=1200)
args = ap.parse_args()
f = args.grid / 2048
grid, angles, bins = args.grid, max(2, round(720 * f)), max(2, round(2897 * f))
nthreads = os.cpu_count()
t0 = time.perf_counter()
A, At, m, n, x, b, _ = cb.host_problem(grid, angles, bins, 0, nthreads)
build_s = time.perf_counter() - t0
M = scipy.sparse.csr_matrix((A[2].astype(np.float64), A[1], A[0]), shape=(m, n))
S = cb.sparse_sign(args.ell, m, 8, 7)
op = linops.LinearOperator.from_matrix(M)
cfg = solvers.SolverConfig(maxiter=args.maxiter, sketch_rows=args.ell)
res = solvers.slslu(op, b, cfg, x_true=x, sketch=sketch.SketchOperator(args.ell, m, 7, S))
py = [r.wall_ms / 1e3 for r in res.trace.records]
c = cb.run_slslu(A, At, m, n, b, args.ell, args.maxiter, 1e9, nthreads, S=S)
out = {
    "what": "sLSLU seconds per iteration, k = 1..maxiter, config-4 geometry scaled to grid",
    "grid": grid, "angles": angles, "bins": bins, "nnz": int(A[0][-1]), "ell": args.ell, "maxiter": args.maxiter,
    "host_threads": nthreads,
    "python_reference_s_per_iter": float(np.mean(py)),
    "python_reference_iter_s": [round(v, 4) for v in py],
    "c_port_s_per_iter": float(np.mean(c["iter_s"])),
    "c_port_threads": nthreads,
    "python_over_c_port": float(np.mean(py) / np.mean(c["iter_s"])),
    "nnz_full_cfg4": 3845024720,
    "python_reference_full_size_estimate_s_per_iter": float(np.mean(py) * 3845024720 / int(A[0][-1])),
    "note": "full-size estimate scales the measured time by the nonzero count (csr_matvec is single-threaded and "
            "dominates); the Python reference cannot build the full config-4 operator on a 62 GB host",
    "operator_build_s": build_s,
}
os.makedirs(os.path.join(ROOT, "profiles", "r2"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", "r2", "reference_python_scaled.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out, indent=1))
