"""Apply the device Gaussian sketch a few times (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2502_02721_b200 as hs
m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 600
g = hs.GaussianSketch(ell, m, seed=1)
v = np.random.default_rng(0).random(m).astype(np.float32)
for _ in range(3):
    g.apply(v, np.float32)
print("ok")
