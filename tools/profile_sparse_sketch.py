"""Apply the sparse-sign sketch at config-4 size (ell=1200 rows, m=2,085,840
rays, zeta=8) a few times and check it against its materialised CSR (for ncu:
the launch list gives the tile-partial and reduce kernel durations)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2502_02721_b200 as hs

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2085840
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 1200
t0 = time.perf_counter()
S = hs.SparseSignSketch(ell, m, seed=3, zeta=8)
print(f"create {time.perf_counter() - t0:.2f} s", flush=True)
v = np.random.default_rng(0).standard_normal(m).astype(np.float32)
z = None
for _ in range(5):
    z = S.apply(v, np.float32)
ref = S.materialize() @ v.astype(np.float64)
err = np.abs(z - ref).max() / np.abs(ref).max()
print(f"max rel err vs CSR: {err:.3e}")
assert err < 1e-12
z2 = S.apply(v, np.float32)
assert np.array_equal(z, z2), "not deterministic"
print("ok")
