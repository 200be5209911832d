"""P-rank row-sharded solves on one GPU (hs_comm_init_local: P contexts, one
host thread per rank, collectives as stream-ordered device copies between the
contexts -- the NCCL path's partition and message sequence).  For P = 2, 4, 8
the sharded loops of hs_dist.inc must reproduce the single-GPU path bit for
bit: pivots, H, W, the basis shards, the sketched columns Z, y, x and the
sketched residuals (every output entry of A l and A^T d is summed
on one rank in reference order, and the sketches sum the same granule/tile
partials in the same global order for any P)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib

    _lib.load()  # fail loudly if the extension is missing
    return hs


def _ranks(P, fn):
    from paper_2502_02721_b200 import dist as hsd

    ctxs = hsd.local_group(P)
    try:
        return hsd.run_ranks(fn, ctxs)
    finally:
        for c in ctxs:
            c.close()


def _same(r1, rp, rect):
    f1, fp = r1.factorization, rp.factorization
    assert rp.termination == r1.termination
    np.testing.assert_array_equal(fp.t, f1.t)
    if rect:
        np.testing.assert_array_equal(fp.g, f1.g)
        np.testing.assert_array_equal(fp.W_matrix(), f1.W_matrix())
    np.testing.assert_array_equal(fp.H_matrix(), f1.H_matrix())
    np.testing.assert_array_equal(fp._res.Z, f1._res.Z)
    np.testing.assert_array_equal(fp._res.y, f1._res.y)
    np.testing.assert_array_equal(rp.x, r1.x)
    for col in ("sres_norm", "proj_obj", "matvecs", "tmatvecs", "sketches"):
        assert rp.trace.column(col) == r1.trace.column(col), col
    # rel_err: the squared-error partials are summed per rank, then over ranks;
    # with a Gaussian S1 the single-GPU loop sketches in batches, so its late
    # iterates' errors come from the fp64 x pass instead of the fused (fp32-
    # accumulated) one -- equal to rounding, not bitwise
    np.testing.assert_allclose(rp.trace.column("rel_err"), r1.trace.column("rel_err"), rtol=1e-6)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("lam,basis", [(0.0, "float32"), (1e-3, "float32")])
def test_local_ranks_slslu_bitwise(hs, P, lam, basis):
    """Row-sharded sLSLU on the tomography operator (all-gathers of l_k and
    d_{k+1}, owner-picked pivot rows, merged argmax candidates, all-gathered
    sketch partials) on P in-process ranks == the single-GPU solve."""
    from paper_2502_02721_b200 import dist as hsd
    from paper_2502_02721_b200.problems import add_noise, random_ellipses

    grid, angles, bins, K = 64, 64, 91, 30
    x = random_ellipses(grid, 10, 0).ravel()
    cfg = hs.SolverConfig(maxiter=K, lam=lam, dtype="float32", basis_dtype=basis, sketch_kind="gaussian")
    op1 = hs.TomographyOperator(grid, angles, bins, dtype=np.float32)
    b, _ = add_noise(op1.matvec(x), 0.01, 1)
    S = hs.SparseSignSketch(4 * K, op1.rows, seed=2, zeta=8)
    sk = hs.SketchOperator(4 * K, op1.rows, 2, S)
    r1 = hs.slslu(op1, b, cfg, x_true=x, sketch=sk)
    L1, D1 = r1.factorization.L_matrix(), r1.factorization.D_matrix()

    def rank(r, ctx):
        op = hs.TomographyOperator(grid, angles, bins, dtype=np.float32)
        np.testing.assert_array_equal(op.matvec(x), op1.matvec(x))
        res = hs.slslu(op, b, cfg, x_true=x, sketch=sk)
        pl = hsd.shard_plan(grid, angles, bins, P, r)
        f = res.factorization
        np.testing.assert_array_equal(f.L_matrix(), L1[pl.n_off:pl.n_off + pl.n_loc])
        np.testing.assert_array_equal(f.D_matrix(), D1[pl.m_off:pl.m_off + pl.m_loc])
        return res

    for rp in _ranks(P, rank):
        _same(r1, rp, True)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("basis,lam", [("float32", 0.0), ("bfloat16", 0.0), ("float32", 0.05)])
def test_local_ranks_scmrh_psf_bitwise(hs, P, basis, lam):
    """Row-sharded sCMRH on the PSF operator (halo exchange of kh/2 rows with
    each neighbour, batched Gaussian sketches with all-gathered partials) on P
    in-process ranks == the single-GPU solve."""
    from paper_2502_02721_b200 import dist as hsd
    from paper_2502_02721_b200.problems import add_noise, gaussian_psf, rectangles_and_discs

    K, size = 30, 128
    psf = gaussian_psf(2.0, radius=7)
    x = rectangles_and_discs(size, 20, 0).ravel()
    op1 = hs.PsfOperator(size, psf, dtype=np.float32)
    b, _ = add_noise(op1.matvec(x), 0.01, 1)
    cfg = hs.SolverConfig(maxiter=K, sketch_rows=4 * K, dtype="float32", basis_dtype=basis, sketch_kind="gaussian",
                          lam=lam)
    solve = hs.scmrh_tikhonov if lam > 0 else hs.scmrh
    r1 = solve(op1, b, cfg, x_true=x)
    L1 = r1.factorization.L_matrix()

    def rank(r, ctx):
        op = hs.PsfOperator(size, psf, dtype=np.float32)
        res = solve(op, b, cfg, x_true=x)
        pl = hsd.psf_shard_plan(size, size, P, r)
        np.testing.assert_array_equal(res.factorization.L_matrix(), L1[pl.n_off:pl.n_off + pl.n_loc])
        return res

    for rp in _ranks(P, rank):
        _same(r1, rp, False)


def test_local_ranks_failure_releases_peers(hs):
    """A rank that fails before a collective releases its peers (no hang)."""
    from paper_2502_02721_b200.problems import random_ellipses

    grid, angles, bins, K = 64, 64, 91, 10
    x = random_ellipses(grid, 10, 0).ravel()
    cfg = hs.SolverConfig(maxiter=K, dtype="float32", sketch_kind="gaussian")

    def rank(r, ctx):
        op = hs.TomographyOperator(grid, angles, bins, dtype=np.float32)
        b = op.matvec(x)
        if r == 1:
            raise ValueError("rank 1 fails before the solve")
        return hs.slslu(op, b, cfg, x_true=x)

    with pytest.raises((ValueError, RuntimeError)):
        _ranks(2, rank)


def test_nccl_bindings_single_rank(hs):
    """The run-time NCCL bindings (dlopen'ed libnccl.so.2: all-gather, fp64 sum
    all-reduce, grouped send/recv -- every call hs_dist.inc makes) on a one-rank
    communicator: results checked inside the library.  Two ranks cannot share
    one GPU under NCCL, so the P-rank data path itself is covered by the
    in-process ranks above."""
    from paper_2502_02721_b200 import dist as hsd

    hsd.nccl_selftest()
