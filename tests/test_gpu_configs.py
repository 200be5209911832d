"""Full-size parity on BASELINE configs 1-3: the device solve (through the C
ABI) against the CPU oracle on the same operator, b and sketch matrices.

Configs 4 and 5 exceed the numpy oracle (a 3.8e9-nonzero CSR; an 80 GB
Gaussian S).  Config 4 (the metric config) is checked against the C port of
the reference loop (oracle/coracle.c) on the host-built operator with the
same b and the same sketch matrix; config 5 with bf16 basis storage against
the bf16-storage oracle32 at 512^2 (same 31x31 PSF), and its full 4096^2
pivots (fp32 storage) against the C port of the square process.

Bars (north_star): pivot sequences bit-exact, H / W and the bases bit-exact;
fp32 (configs 2, 3) sres, proj_obj, rel_err and x within 1e-4 relative;
fp64 (config 1) within 1e-10 relative for the first 30 iterations and, over
the whole run, 2e-5: the order of the reference's own sensitivity envelope on
this operator (3.6e-6 on x at k = 100 between two orderings of
the same dense products), since the projected solve here is an incremental
CGS2 QR instead of geqp3 from scratch and at late k the
semi-convergent iterate is ~1e6 x |x_true|.
"""

import os

import numpy as np
import pytest
import scipy.sparse

pytestmark = pytest.mark.gpu

from oracle import hessketch_oracle as ho  # noqa: E402
from oracle import tomo_oracle as to  # noqa: E402


@pytest.fixture(scope="module")
def hs():
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib

    _lib.load()  # fail loudly if the extension is missing
    return hs


def _rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _column(ref, name):
    return np.array(ref.column(name), dtype=float)


def _check_trace(res, ref, rtol, k_tight=None, rtol_tight=None):
    for name in ("sres_norm", "proj_obj", "rel_err"):
        dev, ora = res.trace.column(name), _column(ref, name)
        assert len(dev) == len(ora)
        if k_tight:
            np.testing.assert_allclose(dev[:k_tight], ora[:k_tight], rtol=rtol_tight, err_msg=name)
        np.testing.assert_allclose(dev, ora, rtol=rtol, err_msg=name)
    assert res.termination == ref.termination
    for name in ("matvecs", "tmatvecs", "sketches"):
        assert list(res.trace.column(name)) == list(ref.column(name)), name


def test_config1_dense_fp64(hs):
    from paper_2502_02721_b200.problems import make_workload, toeplitz_blur_1d

    w = make_workload(1)
    M = toeplitz_blur_1d(1024)  # the matrix make_workload(1) uploads
    res = hs.scmrh(w.operator, w.b, w.cfg, x_true=w.x_true)
    # the reference draw of S (PCG64, sketch.py:43-53) is what the oracle draws with S2=None
    ref = ho.hessenberg_solve(ho.dense_operator(M, np.float64, sequential=True), w.b, square=True,
                              maxiter=w.cfg.maxiter, ell=w.cfg.sketch_rows, seed=w.cfg.seed, x_true=w.x_true)
    t_ref, _ = ho.pivots_of(ref.state)
    st = res.factorization
    np.testing.assert_array_equal(st.t[: len(t_ref)], t_ref)
    np.testing.assert_array_equal(st.H_matrix(), ref.state.H_matrix())
    np.testing.assert_array_equal(st.L_matrix(), np.column_stack(ref.state.L))
    # late iterations: semi-convergence has blown x up to ~1e6 x |x_true| and the
    # projected system is nearly singular; measured 6.0e-6 on rel_err, 4e-6 on x
    _check_trace(res, ref, rtol=2e-5, k_tight=30, rtol_tight=1e-10)
    assert _rel(res.x, ref.x) <= 2e-5


def test_config2_psf_fp32(hs):
    from paper_2502_02721_b200.problems import gaussian_psf, make_workload

    w = make_workload(2)
    size = w.meta["image"][0]
    psf = gaussian_psf(2.0, radius=7)
    gs = hs.GaussianSketch(w.cfg.sketch_rows, size * size, seed=w.cfg.seed)
    res = hs.scmrh(w.operator, w.b, w.cfg, x_true=w.x_true,
                   sketch=hs.SketchOperator(w.cfg.sketch_rows, size * size, w.cfg.seed, gs))
    A = ho.Operator(size * size, size * size,
                    lambda v: to.psf_stencil(v.reshape(size, size), psf, False, np.float32).ravel(),
                    lambda v: to.psf_stencil(v.reshape(size, size), psf, True, np.float32).ravel(), np.float32)
    ref = ho.hessenberg_solve(A, w.b, square=True, maxiter=w.cfg.maxiter, S2=gs.materialize(), x_true=w.x_true)
    t_ref, _ = ho.pivots_of(ref.state)
    st = res.factorization
    np.testing.assert_array_equal(st.t[: len(t_ref)], t_ref)
    np.testing.assert_array_equal(st.H_matrix(), ref.state.H_matrix())
    _check_trace(res, ref, rtol=1e-4)
    assert _rel(res.x, ref.x) <= 1e-4


def test_config3_tomography_fp32_tikhonov(hs):
    import os

    from oracle import cpu_baseline as cb
    from paper_2502_02721_b200.problems import make_workload

    w = make_workload(3)
    grid, angles, bins = w.meta["grid"], w.meta["angles"], w.meta["bins"]
    (rp, ci, cv), _, m, n = cb.host_tomography(grid, angles, bins, os.cpu_count())
    K = scipy.sparse.csr_matrix((cv, ci, rp), shape=(m, n))
    assert K.nnz == w.meta["nnz"]
    ell, seed = w.cfg.sketch_rows, w.cfg.seed
    # S1 as the device realises it for sketch_kind="gaussian" (solvers.py:316)
    S1 = hs.GaussianSketch(ell, n, hs.derive_seed(seed, 1))
    res = hs.slslu(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    ref = ho.hessenberg_solve(ho.csr_operator(K, np.float32), w.b, square=False, maxiter=w.cfg.maxiter,
                              S2=w.sketch.entries.materialize(), S1=S1.materialize(), lam=w.cfg.lam,
                              x_true=w.x_true)
    t_ref, g_ref = ho.pivots_of(ref.state)
    st = res.factorization
    np.testing.assert_array_equal(st.t[: len(t_ref)], t_ref)
    np.testing.assert_array_equal(st.g[: len(g_ref)], g_ref)
    np.testing.assert_array_equal(st.H_matrix(), ref.state.H_matrix())
    np.testing.assert_array_equal(st.W_matrix(), ref.state.W_matrix())
    _check_trace(res, ref, rtol=1e-4)
    assert _rel(res.x, ref.x) <= 1e-4


def test_config4_solve_vs_c_port(hs):
    """Config 4 (the metric config: 2048^2 tomography, 720 x 2897 rays, 3.85e9
    nonzeros, sparse-sign S2 with ell = 1200) at full size, 100 sLSLU
    iterations (all 300 with HS_FULL_PARITY=1: profiles/r2/parity_cfg4_300.txt):
    the device solve against oracle/coracle.c (the C port of
    solvers.py:410-539 with hessenberg.py:329-390) on the host-built operator,
    the same b and the materialised device S2.  Pivots t and g bit-exact at
    every iteration; sres and x within the north-star fp32 bar 1e-4."""
    from oracle import cpu_baseline as cb
    from paper_2502_02721_b200.problems import make_workload

    K = 300 if os.environ.get("HS_FULL_PARITY") else 100
    w = make_workload(4, maxiter=K)
    res = hs.slslu(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=w.sketch)
    assert res.termination == "maxiter" and len(res.trace.records) == K
    S = w.sketch.entries.materialize()
    nthreads = os.cpu_count()
    A, At, m, n = cb.host_tomography(w.meta["grid"], w.meta["angles"], w.meta["bins"], nthreads)
    assert int(A[0][-1]) == w.meta["nnz"]
    c = cb.run_slslu(A, At, m, n, w.b, w.cfg.sketch_rows, K, 1e9, nthreads, S=S)
    del A, At
    assert c["done"] == K
    f = res.factorization
    np.testing.assert_array_equal(f.t[: K + 1], c["t"][: K + 1])
    np.testing.assert_array_equal(f.g[: K + 1], c["g"][: K + 1])
    np.testing.assert_allclose(res.trace.column("sres_norm"), c["sres"], rtol=1e-4)
    assert _rel(res.x, c["x"]) < 1e-4


def test_config5_bf16_storage_vs_oracle32(hs):
    """Config 5's arithmetic (31x31 PSF, sigma 4; bf16 basis storage, fp32
    pivoting / elimination / normalisation; Gaussian S2, ell = 600) at 512^2,
    40 sCMRH iterations, against oracle32 with bf16 storage (each stored
    column rounded to nearest-even bf16; the elimination and the operator read
    the stored values) on the same b and the materialised device S2: pivots
    and H bit-exact; sres, proj_obj, rel_err and x within 1e-4."""
    from paper_2502_02721_b200.problems import gaussian_psf, make_workload

    K = 40
    w = make_workload(5, scale=512, maxiter=K)
    assert w.cfg.basis_dtype == "bfloat16"
    size = w.meta["image"][0]
    psf = gaussian_psf(4.0, radius=15)
    S = hs.GaussianSketch(w.cfg.sketch_rows, size * size, seed=3)
    res = hs.scmrh(w.operator, w.b, w.cfg, x_true=w.x_true, sketch=hs.SketchOperator(S.out_rows, S.in_rows, 3, S))
    A = ho.Operator(size * size, size * size,
                    lambda v: to.psf_stencil(v.reshape(size, size), psf, False, np.float32).ravel(),
                    lambda v: to.psf_stencil(v.reshape(size, size), psf, True, np.float32).ravel(), np.float32)
    ref = ho.hessenberg_solve(A, w.b, square=True, maxiter=K, S2=S.materialize(), x_true=w.x_true,
                              storage="bfloat16")
    t_ref, _ = ho.pivots_of(ref.state)
    f = res.factorization
    np.testing.assert_array_equal(f.t[: len(t_ref)], t_ref)
    np.testing.assert_array_equal(f.H_matrix(), ref.state.H_matrix())
    # the stored basis itself (bf16 values)
    np.testing.assert_array_equal(f.L_matrix()[:, :8], np.column_stack(ref.state.L[:8]).astype(np.float64))
    _check_trace(res, ref, 1e-4)
    assert _rel(res.x, ref.x) < 1e-4


def test_config5_fullsize_pivots_vs_c_port(hs):
    """Config 5 at its full 4096^2 size (16.8M unknowns, 31x31 PSF), fp32
    basis storage: all 150 pivots and Hessenberg columns of the
    device sCMRH bit-exact against the C port of the square process
    (hessenberg.py:160-226) with the order-specified stencil.  Pivots do not
    depend on the sketch, so no 80 GB S is needed.  Also the
    full-size operator bit for bit."""
    import dataclasses

    from oracle import cpu_baseline as cb
    from paper_2502_02721_b200.problems import gaussian_psf, make_workload

    K = 150
    w = make_workload(5, maxiter=K)
    cfg = dataclasses.replace(w.cfg, basis_dtype="float32")
    size = w.meta["image"][0]
    psf = gaussian_psf(4.0, radius=15)
    img = np.random.default_rng(5).standard_normal(size * size).astype(np.float32)
    np.testing.assert_array_equal(w.operator.matvec(img, np.float32),
                                  cb.psf_conv(img.reshape(size, size), psf).ravel())
    res = hs.scmrh(w.operator, w.b, cfg, x_true=w.x_true)
    t_c, H_c = cb.scmrh_psf_pivots((size, size), psf, w.b, K)
    assert len(t_c) == K + 1
    f = res.factorization
    np.testing.assert_array_equal(f.t[: K + 1], t_c)
    np.testing.assert_array_equal(f.H_matrix(), H_c)
