"""Pin the CPU oracle (oracle/) to fixtures produced by the unmodified reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest
import scipy.signal
import scipy.sparse

from oracle import hessketch_oracle as ho
from oracle import tomo_oracle as to


def _csr(g, prefix="A_"):
    shape = tuple(int(s) for s in g[prefix + "shape"])
    return scipy.sparse.csr_matrix((g[prefix + "data"], g[prefix + "indices"], g[prefix + "indptr"]), shape=shape)


def _check_result(res, g, prefix="", exact=True, rtol=0.0):
    assert res.termination == str(g[prefix + "termination"])
    n = len(res.records)
    assert n == len(g[prefix + "sres_norm"])
    for name in ("matvecs", "tmatvecs", "dots", "sketches"):
        assert [r[name] for r in res.records] == list(g[prefix + name]), name
    assert [r["rank_fallback"] for r in res.records] == list(g[prefix + "rank_fallback"])
    for name in ("sres_norm", "proj_obj", "rel_err"):
        got = np.array([np.nan if r[name] is None else r[name] for r in res.records])
        want = g[prefix + name]
        if exact:
            np.testing.assert_array_equal(got, want, err_msg=name)
        else:
            np.testing.assert_allclose(got, want, rtol=rtol, err_msg=name)
    if exact:
        np.testing.assert_array_equal(res.x, g[prefix + "x"])
    else:
        np.testing.assert_allclose(res.x, g[prefix + "x"], rtol=rtol, atol=rtol * np.abs(g[prefix + "x"]).max())
    st = res.state
    if st is not None and prefix + "t" in g:
        t, gg = ho.pivots_of(st)
        np.testing.assert_array_equal(t, g[prefix + "t"])
        if gg is not None:
            np.testing.assert_array_equal(gg, g[prefix + "g"])
        if exact:
            np.testing.assert_array_equal(st.H_matrix(), g[prefix + "H"])


def test_pivot_hand_examples():
    # hessenberg.py:93-115 semantics, reference tests test_hessenberg.py:135-193
    v = np.array([3.0, -5.0, 2.0])
    assert ho.pivot_full(v, [0, 1, 2]) == (1, -5.0)
    assert ho.pivot_full(v, [0, 2]) == (0, 3.0)
    v = np.array([2.0, -2.0, 2.0])
    assert ho.pivot_full(v, [2, 1, 0]) == (0, 2.0)
    assert ho.pivot_full(v, [2, 1]) == (1, -2.0)
    assert ho.pivot_full(np.zeros(4), [1, 3])[1] == 0.0
    with pytest.raises(ValueError):
        ho.pivot_full(np.ones(3), [])


def test_steps_dense_bitwise(golden):
    g = golden("steps_dense")
    A = ho.dense_operator(g["sq_M"], sequential=False)
    st = ho.init_square(A, g["sq_b"])
    for _ in range(9):
        ho.step_square(st, A)
    np.testing.assert_array_equal(st.t[: len(st.L)], g["sq_t"])
    np.testing.assert_array_equal(st.H_matrix(), g["sq_H"])
    np.testing.assert_array_equal(np.column_stack(st.L), g["sq_L"])
    for tag in ("tall", "wide"):
        M = g[f"{tag}_M"]
        A = ho.dense_operator(M, sequential=False)
        st = ho.init_generalized(A, g[f"{tag}_b"])
        for _ in range(min(M.shape) + 2):
            if st.breakdown:
                break
            ho.step_generalized(st, A)
        assert st.breakdown == bool(g[f"{tag}_breakdown"])
        assert st.k == int(g[f"{tag}_k"])
        np.testing.assert_array_equal(st.t[: len(st.D)], g[f"{tag}_t"])
        np.testing.assert_array_equal(st.g[: len(st.L)], g[f"{tag}_g"])
        np.testing.assert_array_equal(st.H_matrix(), g[f"{tag}_H"])
        np.testing.assert_array_equal(st.W_matrix(), g[f"{tag}_W"])
        np.testing.assert_array_equal(np.column_stack(st.D), g[f"{tag}_D"])
        np.testing.assert_array_equal(np.column_stack(st.L), g[f"{tag}_L"])


def test_scmrh_dense_bitwise(golden):
    g = golden("scmrh_dense")
    A = ho.dense_operator(g["M"], sequential=False)
    res = ho.hessenberg_solve(A, g["b"], square=True, maxiter=12, seed=5, x_true=g["x_true"])
    _check_result(res, g)
    # the PCG64 draw is the reference's
    np.testing.assert_array_equal(ho.gaussian_sketch_entries(130, 40, 5), g["S2"])
    res = ho.hessenberg_solve(A, g["b"], square=True, maxiter=8, S2=g["S2_orth"], x_true=g["x_true"])
    _check_result(res, g, "orth_")
    res = ho.hessenberg_solve(A, g["b"], square=True, maxiter=6, seed=2, x0=g["x0"])
    _check_result(res, g, "x0_")
    res = ho.hessenberg_solve(A, g["b"], square=True, maxiter=7, seed=3, lam=0.4)
    _check_result(res, g, "tik_")


def test_slslu_dense_bitwise(golden):
    g = golden("slslu_dense")
    A = ho.dense_operator(g["M"], sequential=False)
    res = ho.hessenberg_solve(A, g["b"], square=False, maxiter=10, seed=7, x_true=g["x_true"])
    _check_result(res, g)
    res = ho.hessenberg_solve(A, g["b"], square=False, maxiter=9, seed=3, lam=0.7, x_true=g["x_true"])
    _check_result(res, g, "tik_")
    np.testing.assert_array_equal(ho.gaussian_sketch_entries(100, 25, ho.derive_seed(3, 1)), g["S1_tik"])
    Aw = ho.dense_operator(g["Mw"], sequential=False)
    res = ho.hessenberg_solve(Aw, g["bw"], square=False, maxiter=9, seed=1)
    _check_result(res, g, "w_")
    Ah = ho.dense_operator(g["Mh"], sequential=False)
    res = ho.hessenberg_solve(Ah, np.array([1.0, 3.0]), square=False, maxiter=1, seed=0)
    _check_result(res, g, "h_")


def test_dense_sequential_order_keeps_pivots(golden):
    """The oracle pins dense A@x to a sequential row order (what the device
    computes); against the reference's BLAS order the pivots must not move and
    the iterates agree to rounding."""
    g = golden("scmrh_dense")
    A = ho.dense_operator(g["M"], sequential=True)
    res = ho.hessenberg_solve(A, g["b"], square=True, maxiter=12, seed=5, x_true=g["x_true"])
    _check_result(res, g, exact=False, rtol=1e-9)


def test_tomography_matrix_bitwise(golden):
    g = golden("tomo_matrices")
    for grid, angles in ((8, 6), (13, 7), (16, 12)):
        want = _csr(g, f"tomo{grid}x{angles}_")
        got = to.tomography_matrix(grid, angles)
        np.testing.assert_array_equal(got.indptr, want.indptr)
        np.testing.assert_array_equal(got.indices, want.indices)
        np.testing.assert_array_equal(got.data, want.data)


def test_csr_matvec_is_sequential(golden):
    """scipy csr_matvec == left-to-right, no-FMA row sum (float64 and float32)."""
    g = golden("tomo_matrices")
    M = _csr(g, "tomo16x12_")
    rng = np.random.default_rng(0)
    for dt in (np.float64, np.float32):
        x = rng.standard_normal(M.shape[1]).astype(dt)
        Md = M.astype(dt)
        got = to.csr_sequential_matvec(Md.indptr, Md.indices, Md.data, x, dt)
        np.testing.assert_array_equal(got, Md @ x)


def test_slslu_tomo_bitwise(golden):
    g = golden("slslu_tomo16")
    K = _csr(g)
    S2 = _csr(g, "S2_")
    A = ho.csr_operator(K)
    res = ho.hessenberg_solve(A, g["b"], square=False, maxiter=40, S2=S2, x_true=g["x_true"])
    _check_result(res, g)
    res = ho.hessenberg_solve(A, g["b"], square=False, maxiter=30, S2=S2, lam=1e-3, seed=11, x_true=g["x_true"])
    _check_result(res, g, "tik_")


def test_psf_stencil_matches_scipy(golden):
    g = golden("scmrh_deblur16")
    img = g["img"]
    conv = to.psf_stencil(img, g["psf"], transpose=False)
    corr = to.psf_stencil(img, g["psf"], transpose=True)
    scale = np.abs(g["conv"]).max()
    assert np.abs(conv.ravel() - g["conv"]).max() <= 1e-14 * scale
    assert np.abs(corr.ravel() - g["corr"]).max() <= 1e-14 * scale
    # direct check against scipy for a non-square kernel too
    K = np.random.default_rng(1).random((3, 5))
    assert np.allclose(to.psf_stencil(img, K), scipy.signal.convolve2d(img, K, mode="same"), rtol=1e-14, atol=1e-14)
    assert np.allclose(to.psf_stencil(img, K, True), scipy.signal.correlate2d(img, K, mode="same"), rtol=1e-14, atol=1e-14)


def test_scmrh_deblur_stencil_vs_reference(golden):
    """Tap-ordered stencil injected into the oracle: pivots identical to the
    reference's convolve2d run, iterates within rounding."""
    g = golden("scmrh_deblur16")
    size = int(g["size"])
    psf = g["psf"]
    A = ho.Operator(size * size, size * size,
                    lambda v: to.psf_stencil(v.reshape(size, size), psf).ravel(),
                    lambda v: to.psf_stencil(v.reshape(size, size), psf, True).ravel())
    res = ho.hessenberg_solve(A, g["b"], square=True, maxiter=25, seed=6, x_true=g["x_true"])
    _check_result(res, g, exact=False, rtol=1e-7)


def test_edge_cases(golden):
    g = golden("edge_cases")
    res = ho.hessenberg_solve(ho.identity_operator(5), g["id_b"], square=True, maxiter=3, seed=42)
    _check_result(res, g, "id_")
    res = ho.hessenberg_solve(ho.dense_operator(np.ones((4, 3))), np.zeros(4), square=False, maxiter=2)
    assert res.termination == str(g["zero_termination"]) == "trivial"
    np.testing.assert_array_equal(res.x, g["zero_x"])
    res = ho.hessenberg_solve(ho.dense_operator(np.array([[1.0], [0.0]])), np.array([0.0, 1.0]), square=False, maxiter=2)
    assert res.termination == str(g["ne_termination"]) == "trivial"
    res = ho.hessenberg_solve(ho.dense_operator(g["tie_M"], sequential=False), g["tie_b"], square=True, maxiter=3, seed=1)
    _check_result(res, g, "tie_")


def test_validation_errors():
    A = ho.dense_operator(np.eye(8) * 2.0)
    with pytest.raises(ValueError):
        ho.hessenberg_solve(A, np.ones(8), square=True, maxiter=6, ell=4)
    with pytest.raises(ValueError):
        ho.hessenberg_solve(ho.dense_operator(np.ones((3, 2))), np.ones(3), square=True, maxiter=2)


def test_oracle32_tracks_oracle64(golden):
    """The fp32 restatement keeps the fp64 pivot sequence on a well-separated
    problem and its iterates agree to fp32 accuracy."""
    g = golden("slslu_tomo16")
    K = _csr(g)
    S2 = _csr(g, "S2_")
    r64 = ho.hessenberg_solve(ho.csr_operator(K), g["b"], square=False, maxiter=10, S2=S2, x_true=g["x_true"])
    r32 = ho.hessenberg_solve(ho.csr_operator(K, np.float32), g["b"], square=False, maxiter=10, S2=S2, x_true=g["x_true"])
    t64, g64 = ho.pivots_of(r64.state)
    t32, g32 = ho.pivots_of(r32.state)
    np.testing.assert_array_equal(t64, t32)
    np.testing.assert_array_equal(g64, g32)
    np.testing.assert_allclose(r32.x, r64.x, rtol=1e-3, atol=1e-4 * np.abs(r64.x).max())


def test_sampled_pivoting_and_unsketched_bitwise(golden):
    """Sampled pivoting (hessenberg.py:93-124, rng.choice over the swap-ordered
    admissible list, full-scan fallback on an all-zero sample) and the
    unsketched cmrh / lslu (solvers.py:542-559) against the reference."""
    g = golden("sampled_unsketched")
    A = ho.dense_operator(g["sq_M"], sequential=False)
    b, xt = g["sq_b"], g["sq_x_true"]
    res = ho.hessenberg_solve(A, b, square=True, maxiter=15, seed=5, x_true=xt, pivot_sample=5, pivot_seed=13)
    _check_result(res, g, "samp_sq_")
    res = ho.hessenberg_solve(A, b, square=True, maxiter=15, x_true=xt, sketched=False)
    _check_result(res, g, "cmrh_")
    res = ho.hessenberg_solve(A, b, square=True, maxiter=12, lam=0.3, x_true=xt, sketched=False)
    _check_result(res, g, "cmrh_tik_")
    Ab = ho.dense_operator(g["band_M"], sequential=False)
    res = ho.hessenberg_solve(Ab, g["band_b"], square=True, maxiter=10, sketched=False, pivot_sample=3, pivot_seed=4)
    _check_result(res, g, "band_")
    Ar = ho.dense_operator(g["re_M"], sequential=False)
    b, xt = g["re_b"], g["re_x_true"]
    res = ho.hessenberg_solve(Ar, b, square=False, maxiter=12, seed=7, x_true=xt, pivot_sample=4, pivot_seed=2)
    _check_result(res, g, "samp_re_")
    res = ho.hessenberg_solve(Ar, b, square=False, maxiter=12, x_true=xt, sketched=False)
    _check_result(res, g, "lslu_")
    res = ho.hessenberg_solve(Ar, b, square=False, maxiter=10, lam=0.5, x_true=xt, sketched=False)
    _check_result(res, g, "lslu_tik_")
    res = ho.hessenberg_solve(Ar, b, square=False, maxiter=10, x_true=xt, sketched=False, pivot_sample=6, pivot_seed=1)
    _check_result(res, g, "lslu_samp_")
    K = _csr(golden("tomo_matrices"), "tomo16x12_")
    At = ho.csr_operator(K)
    S2 = _csr(g, "tomo_S2_")
    res = ho.hessenberg_solve(At, g["tomo_b"], square=False, maxiter=30, S2=S2, x_true=g["tomo_x_true"],
                              pivot_sample=25, pivot_seed=8)
    _check_result(res, g, "tomo_samp_")
    res = ho.hessenberg_solve(At, g["tomo_b"], square=False, maxiter=30, x_true=g["tomo_x_true"], sketched=False)
    _check_result(res, g, "tomo_lslu_")


def test_rank_fallback_bitwise(golden):
    """Low-rank operators: pivoted-QR rank gate and lstsq minimum-norm fallback
    from the first deficient iteration on (solvers.py:204-218)."""
    g = golden("rank_fallback")
    A = ho.csr_operator(scipy.sparse.csr_matrix(g["sq_M"]))
    res = ho.hessenberg_solve(A, g["sq_b"], square=True, maxiter=8, seed=1, ell=40, x_true=g["sq_xt"])
    _check_result(res, g, "sq_")
    res = ho.hessenberg_solve(A, g["sq_b"], square=True, maxiter=8, x_true=g["sq_xt"], sketched=False)
    _check_result(res, g, "cm_")
    Ar = ho.csr_operator(scipy.sparse.csr_matrix(g["re_M"]))
    res = ho.hessenberg_solve(Ar, g["re_b"], square=False, maxiter=9, seed=3, ell=40, x_true=g["sq_xt"])
    _check_result(res, g, "re_")
    res = ho.hessenberg_solve(Ar, g["re_b"], square=False, maxiter=9, x_true=g["sq_xt"], sketched=False)
    _check_result(res, g, "ll_")


def test_printed_f_variant_bitwise(golden):
    """slslu_tikhonov(printed_f_columns=True) (solvers.py:460-461, 488-490)."""
    g = golden("printed_f")
    A = ho.dense_operator(g["M"], sequential=False)
    res = ho.hessenberg_solve(A, g["b"], square=False, maxiter=8, seed=6, lam=0.5, x_true=g["xt"], printed_f=True)
    _check_result(res, g, "pr_")
    res = ho.hessenberg_solve(A, g["b"], square=False, maxiter=8, seed=6, lam=0.5, x_true=g["xt"])
    _check_result(res, g, "df_")
    assert not np.allclose(g["pr_x"], g["df_x"])


def _check_krylov(res, g, prefix):
    assert res.termination == str(g[prefix + "termination"])
    assert len(res.records) == len(g[prefix + "proj_obj"])
    for name in ("matvecs", "tmatvecs", "dots", "sketches"):
        assert [r[name] for r in res.records] == list(g[prefix + name]), name
    for name in ("proj_obj", "rel_err"):
        got = np.array([np.nan if r[name] is None else r[name] for r in res.records])
        np.testing.assert_array_equal(got, g[prefix + name], err_msg=name)
    if prefix + "res_norm" in g:
        np.testing.assert_array_equal([r["res_norm"] for r in res.records], g[prefix + "res_norm"])
    np.testing.assert_array_equal(res.x, g[prefix + "x"])


def test_gmres_lsqr_bitwise(golden):
    """The comparison solvers restated (solvers.py:256-403): counters including
    the tracked inner products, x, proj_obj, rel_err, res_norm bit for bit."""
    g = golden("krylov")
    A = ho.dense_operator(g["sq_M"], sequential=False)
    b, xt = g["sq_b"], g["sq_x_true"]
    _check_krylov(ho.gmres(A, b, maxiter=15, x_true=xt, diagnostics=True), g, "gm_")
    _check_krylov(ho.gmres(A, b, maxiter=12, lam=0.3, x_true=xt), g, "gm_tik_")
    _check_krylov(ho.gmres(A, b, maxiter=8, x0=g["x0"], diagnostics=True), g, "gm_x0_")
    _check_krylov(ho.gmres(ho.identity_operator(3), np.array([3.0, -5.0, 2.0]), maxiter=30), g, "gm_id_")
    Ar = ho.dense_operator(g["re_M"], sequential=False)
    b, xt = g["re_b"], g["re_x_true"]
    _check_krylov(ho.lsqr(Ar, b, maxiter=15, x_true=xt, diagnostics=True), g, "ls_")
    _check_krylov(ho.lsqr(Ar, b, maxiter=10, lam=0.5, x_true=xt), g, "ls_tik_")
    _check_krylov(ho.lsqr(Ar, b, maxiter=8, x0=g["x0r"]), g, "ls_x0_")
    _check_krylov(ho.lsqr(ho.dense_operator(g["w_M"], sequential=False), g["w_b"], maxiter=6), g, "ls_w_")
    t = golden("slslu_tomo16")
    K = _csr(golden("tomo_matrices"), "tomo16x12_")
    _check_krylov(ho.lsqr(ho.csr_operator(K), t["b"], maxiter=30, x_true=t["x_true"], diagnostics=True), g, "ls_tomo_")


def test_bf16_storage_oracle():
    """oracle32 with bf16 basis storage (config 5's device path): the rounding
    is round-to-nearest-even (torch's bfloat16 conversion), the stored basis is
    bf16-representable with exact unit pivots and exact zeros at earlier pivot
    rows, and H is the elimination on the stored columns."""
    import torch

    from oracle import hessketch_oracle as ho

    rng = np.random.default_rng(0)
    a = (rng.standard_normal(20000) * 10.0 ** rng.integers(-20, 20, 20000)).astype(np.float32)
    assert np.array_equal(ho.round_bf16(a), torch.from_numpy(a).to(torch.bfloat16).float().numpy())
    n, K = 200, 12
    M = rng.standard_normal((n, n)).astype(np.float32)
    A = ho.dense_operator(M, np.float32)
    b = rng.standard_normal(n)
    ref = ho.hessenberg_solve(A, b, square=True, maxiter=K, S2=rng.standard_normal((4 * K, n)), storage="bfloat16")
    L = np.column_stack(ref.state.L)
    assert np.array_equal(ho.round_bf16(L), L)
    t, _ = ho.pivots_of(ref.state)
    P = L[t[: L.shape[1]], :]
    assert np.all(np.diag(P) == 1.0) and np.all(np.triu(P, 1) == 0.0)
    # without bf16 storage the same problem keeps fp32 columns (not all bf16-representable)
    ref32 = ho.hessenberg_solve(A, b, square=True, maxiter=K, S2=rng.standard_normal((4 * K, n)))
    assert not np.array_equal(ho.round_bf16(np.column_stack(ref32.state.L)), np.column_stack(ref32.state.L))
