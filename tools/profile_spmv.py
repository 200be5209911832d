"""Apply the cfg4-geometry tomography operator a few times (for ncu).

    python tools/profile_spmv.py [--scale 1024] [--reps 3]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2502_02721_b200 as hs

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=1024)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
f = args.scale / 2048
op = hs.TomographyOperator(args.scale, max(2, round(720 * f)), max(2, round(2897 * f)), dtype=np.float32)
x = np.random.default_rng(0).random(op.cols).astype(np.float32)
y = np.random.default_rng(1).random(op.rows).astype(np.float32)
for _ in range(args.reps):
    op.matvec(x, np.float32)
    op.rmatvec(y, np.float32)
print("nnz", op.info()["nnz"], "ok")
