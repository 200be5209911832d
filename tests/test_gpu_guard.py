"""Out-of-bounds-write check of every kernel family (compute-sanitizer is not
available on the GPU pool): with HS_GUARD=1 each device buffer carries 4 KB
guard bands on both sides, verified when the buffer is released.  A battery of
small solves covering the operators (CSR / SELL encodings incl. the step
codes, PSF stencils,
dense), the fused elimination pass, fsub, pivot commit, normalisation, the
sketches (sparse-sign tiles, Gaussian batches, dense), the cooperative
projected solve, sampled pivoting, the step API, GMRES / LSQR, diagnostics and
the P-rank sharded loops must leave every guard band intact."""

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_no_out_of_bounds_writes(monkeypatch):
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib
    from paper_2502_02721_b200 import dist as hsd
    from paper_2502_02721_b200.hessenberg import PivotStrategy
    from paper_2502_02721_b200.problems import add_noise, gaussian_psf, random_ellipses, rectangles_and_discs

    lib = _lib.load()
    monkeypatch.setenv("HS_GUARD", "1")
    before = lib.hs_guard_violations()

    grid, angles, bins, K = 48, 30, 69, 20
    x = random_ellipses(grid, 10, 0).ravel()
    for dt, basis in (("float32", "float32"), ("float64", "float64"), ("float32", "bfloat16")):
        op = hs.TomographyOperator(grid, angles, bins, dtype=np.float32 if dt == "float32" else np.float64)
        b, _ = add_noise(op.matvec(x), 0.01, 1)
        for kind in ("sparse_sign", "gaussian", "pcg64"):
            cfg = hs.SolverConfig(maxiter=K, lam=1e-3, dtype=dt, basis_dtype=basis, sketch_kind=kind)
            hs.slslu(op, b, cfg, x_true=x)
        cfg = hs.SolverConfig(maxiter=K, dtype=dt, basis_dtype=basis, sketch_kind="gaussian",
                              pivot=PivotStrategy.sampled(50, seed=1), compute_diagnostics=True)
        hs.slslu(op, b, cfg, x_true=x)
        hs.lslu(op, b, hs.SolverConfig(maxiter=K, dtype=dt), x_true=x)
        hs.lsqr(op, b, hs.SolverConfig(maxiter=K, dtype=dt), x_true=x)
    # the step-code encoders and kernels (2-bit on A, 8-bit on A^T), forced on a small operator
    monkeypatch.setenv("HS_C2", "2")
    monkeypatch.setenv("HS_T8", "2")
    for g2, a2, b2 in ((48, 30, 69), (50, 33, 41)):
        opc = hs.TomographyOperator(g2, a2, b2, dtype=np.float32)
        xc = random_ellipses(g2, 10, 0).ravel()
        bc, _ = add_noise(opc.matvec(xc), 0.01, 1)
        hs.slslu(opc, bc, hs.SolverConfig(maxiter=K, dtype="float32"), x_true=xc)
        del opc
    monkeypatch.delenv("HS_C2")
    monkeypatch.delenv("HS_T8")
    size = 64
    psf = gaussian_psf(2.0, radius=7)
    xi = rectangles_and_discs(size, 20, 0).ravel()
    op = hs.PsfOperator(size, psf, dtype=np.float32)
    b, _ = add_noise(op.matvec(xi), 0.01, 1)
    for basis in ("float32", "bfloat16"):
        cfg = hs.SolverConfig(maxiter=K, sketch_rows=4 * K, dtype="float32", basis_dtype=basis,
                              sketch_kind="gaussian")
        hs.scmrh(op, b, cfg, x_true=xi)
        hs.scmrh_tikhonov(op, b, hs.SolverConfig(maxiter=K, sketch_rows=4 * K, lam=0.05, dtype="float32",
                                                  basis_dtype=basis, sketch_kind="gaussian"), x_true=xi)
    hs.gmres(op, b, hs.SolverConfig(maxiter=K, dtype="float32"), x_true=xi)
    M = np.random.default_rng(0).standard_normal((200, 200))
    dop = hs.DenseOperator(M)
    hs.scmrh(dop, M @ np.ones(200), hs.SolverConfig(maxiter=K), x_true=np.ones(200))
    st = hs.init_square(dop, M @ np.ones(200))
    for _ in range(5):
        st = hs.step_square(st, dop)
    # P-rank sharded loops (in-process communicator)
    tomo_b = hs.TomographyOperator(64, 64, 91, dtype=np.float32).matvec(random_ellipses(64, 10, 0).ravel())

    def rank(r, ctx):
        op = hs.TomographyOperator(64, 64, 91, dtype=np.float32)
        cfg = hs.SolverConfig(maxiter=K, lam=1e-3, dtype="float32", sketch_kind="gaussian")
        return hs.slslu(op, tomo_b, cfg).x

    ctxs = hsd.local_group(2)
    try:
        hsd.run_ranks(rank, ctxs)
    finally:
        for c in ctxs:
            c.close()
    del op, dop, st
    gc.collect()
    assert lib.hs_guard_violations() == before
