"""Full-size checks on the GPU (BASELINE configs 3 and 4 at their real sizes):
device operator applications bit-identical to the C port of the reference
CSR matvec on the host-built operator, and size-independent properties of a
short sLSLU run (exact unit-triangular bases at the pivots, A L_k = D_{k+1} H,
deterministic replay).  Slow (host operator build); marked gpu."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib

    _lib.load()
    return hs


def _host_matvec(A, x, nthreads):
    from oracle import cpu_baseline as cb

    y = np.empty(len(A[0]) - 1, dtype=np.float32)
    cb.lib().co_spmv_f32_export(len(A[0]) - 1, cb._p(A[0]), cb._p(A[1]), cb._p(A[2]), cb._p(x), cb._p(y), nthreads)
    return y


@pytest.mark.parametrize("cfg", [3, 4])
def test_fullsize_operator_bitwise_vs_c_port(hs, cfg):
    from oracle import cpu_baseline as cb

    grid, angles, bins = (512, 180, 725) if cfg == 3 else (2048, 720, 2897)
    nthreads = os.cpu_count()
    A, At, m, n = cb.host_tomography(grid, angles, bins, nthreads)
    op = hs.TomographyOperator(grid, angles, bins, dtype=np.float32)
    assert op.info()["nnz"] == int(A[0][-1]) == op.info()["nnz_t"]
    rng = np.random.default_rng(cfg)
    x = rng.standard_normal(n).astype(np.float32)
    y = rng.standard_normal(m).astype(np.float32)
    np.testing.assert_array_equal(op.matvec(x, np.float32), _host_matvec(A, x, nthreads))
    np.testing.assert_array_equal(op.rmatvec(y, np.float32), _host_matvec(At, y, nthreads))
    del A, At


def test_fullsize_slslu_properties(hs):
    from paper_2502_02721_b200.problems import make_workload

    w = make_workload(4, maxiter=8)
    r1 = hs.slslu(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    r2 = hs.slslu(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    assert np.array_equal(r1.x, r2.x)  # deterministic replay (test_solvers.py:319-326)
    assert r1.trace.column("sres_norm") == r2.trace.column("sres_norm")
    st = r1.factorization
    D, L = st.D_matrix(), st.L_matrix()
    t, g = st.t[: D.shape[1]], st.g[: L.shape[1]]
    Dt, Lt = D[t, :], L[g, :]
    assert np.all(np.diag(Dt) == 1.0) and np.all(np.triu(Dt, 1) == 0.0)
    assert np.all(np.diag(Lt) == 1.0) and np.all(np.triu(Lt, 1) == 0.0)
    assert len(set(t.tolist())) == len(t) and len(set(g.tolist())) == len(g)
    # A L_k = D_{k+1} H_{k+1,k} through the device operator (fp64 work on the fp32 values)
    k = st.k
    H = st.H_matrix(rows=D.shape[1])
    AL = np.column_stack([w.operator.matvec(L[:, j]) for j in range(k)])
    assert np.linalg.norm(AL - D @ H) <= 1e-5 * np.linalg.norm(AL)
    rel = r1.trace.column("rel_err")
    assert rel[-1] < rel[0]
    assert all(r.dots == 0 for r in r1.trace.records)
