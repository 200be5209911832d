"""Batched Gaussian sketches (hs_sketch.cuh, Solver::run in hs_api.cu).

The basis recurrence never reads a sketch, so the device forms the Gaussian
columns z_k = S2 A l_k (and f_k = S1 l_{k+1}) several iterations at a time with
one pass of the counter-based generator.  These tests pin that the batch size
is invisible: every sketch column, every projected-solve quantity and the
iterate are bit-identical to the per-iteration schedule (HS_SKETCH_BATCH=1),
including partial batches and early breakdown.  rel_err is formed by the
lagged fused pass or, for the last iterations, by a separate fp64 pass, so it
is compared to rounding (1e-12 in fp64, 1e-5 in fp32)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib

    _lib.load()
    return hs


@pytest.mark.parametrize("nv", [1, 3, 8, 11])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_apply_many_bitwise(hs, nv, dtype):
    rng = np.random.default_rng(nv)
    m = 5000
    V = rng.standard_normal((m, nv)).astype(dtype)
    gs = hs.GaussianSketch(72, m, seed=4)
    Z = gs.apply(V, dtype)
    assert Z.shape == (72, nv)
    for w in range(nv):
        np.testing.assert_array_equal(Z[:, w], gs.apply(V[:, w], dtype))
    Sg = gs.materialize()
    np.testing.assert_allclose(Z, Sg @ V.astype(np.float64), rtol=1e-9, atol=1e-9)
    # other kinds go column by column through the same entry point
    ss = hs.SparseSignSketch(40, m, seed=3, zeta=8)
    Zs = ss.apply(V, dtype)
    for w in range(nv):
        np.testing.assert_array_equal(Zs[:, w], ss.apply(V[:, w], dtype))


def _solve_with_batch(monkeypatch, batch, fn):
    monkeypatch.setenv("HS_SKETCH_BATCH", str(batch))
    return fn()


def _same(r1, r2, rel_tol):
    assert r1.termination == r2.termination
    assert len(r1.trace.records) == len(r2.trace.records)
    for col in ("sres_norm", "proj_obj", "matvecs", "tmatvecs", "sketches"):
        assert r1.trace.column(col) == r2.trace.column(col), col
    np.testing.assert_array_equal(r1.x, r2.x)
    np.testing.assert_array_equal(r1.factorization._res.Z, r2.factorization._res.Z)
    np.testing.assert_array_equal(r1.factorization._res.y, r2.factorization._res.y)
    e1, e2 = r1.trace.column("rel_err"), r2.trace.column("rel_err")
    np.testing.assert_allclose(e1, e2, rtol=rel_tol)


@pytest.mark.parametrize("dtype,rel_tol", [("float64", 1e-12), ("float32", 1e-5)])
@pytest.mark.parametrize("maxiter", [8, 21, 40])
def test_batched_deblur_matches_per_iteration(hs, monkeypatch, dtype, rel_tol, maxiter):
    from paper_2502_02721_b200.problems import add_noise, gaussian_psf, rectangles_and_discs

    size = 40
    psf = gaussian_psf(2.0, radius=7)
    x = rectangles_and_discs(size, 20, 0).ravel()
    op = hs.PsfOperator(size, psf, dtype=np.float32 if dtype == "float32" else np.float64)
    b, _ = add_noise(op.matvec(x), 0.01, 1)
    cfg = hs.SolverConfig(maxiter=maxiter, sketch_rows=4 * maxiter + 8, dtype=dtype, sketch_kind="gaussian")
    runs = [_solve_with_batch(monkeypatch, sb, lambda: hs.scmrh(op, b, cfg, x_true=x)) for sb in (1, 8, 3)]
    _same(runs[0], runs[1], rel_tol)
    _same(runs[0], runs[2], rel_tol)


@pytest.mark.parametrize("dtype,rel_tol", [("float64", 1e-12), ("float32", 1e-5)])
def test_batched_tikhonov_tomography_matches_per_iteration(hs, monkeypatch, dtype, rel_tol):
    """sparse-sign S2 with a Gaussian S1 (config 3's shape): the F columns are
    sketched from the stored L columns in batches"""
    from paper_2502_02721_b200.problems import add_noise, random_ellipses

    grid, angles, bins, K = 32, 20, 45, 19
    op = hs.TomographyOperator(grid, angles, bins, dtype=np.float32 if dtype == "float32" else np.float64)
    x = random_ellipses(grid, 10, 0).ravel()
    b, _ = add_noise(op.matvec(x), 0.01, 1)
    ss = hs.SparseSignSketch(100, op.rows, seed=5, zeta=8)
    cfg = hs.SolverConfig(maxiter=K, lam=1e-3, dtype=dtype, sketch_kind="gaussian", sketch_rows=100)
    sk = hs.SketchOperator(100, op.rows, 5, ss)
    runs = [_solve_with_batch(monkeypatch, sb, lambda: hs.slslu(op, b, cfg, x_true=x, sketch=sk)) for sb in (1, 8, 4)]
    _same(runs[0], runs[1], rel_tol)
    _same(runs[0], runs[2], rel_tol)


def test_batched_breakdown_matches_per_iteration(hs, monkeypatch):
    """square 12x12 operator, maxiter past n: full-basis breakdown at k = 12
    inside a batch"""
    rng = np.random.default_rng(3)
    M = rng.standard_normal((12, 12)) + 5 * np.eye(12)
    A = hs.LinearOperator.from_matrix(M)
    b = rng.standard_normal(12)
    x = rng.standard_normal(12)
    cfg = hs.SolverConfig(maxiter=17, sketch_rows=60, sketch_kind="gaussian")
    r1 = _solve_with_batch(monkeypatch, 1, lambda: hs.scmrh(A, b, cfg, x_true=x))
    r8 = _solve_with_batch(monkeypatch, 8, lambda: hs.scmrh(A, b, cfg, x_true=x))
    assert r1.termination == "breakdown"
    _same(r1, r8, 1e-12)
