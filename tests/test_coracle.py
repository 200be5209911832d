"""The C port of the reference loop (oracle/coracle.c, CPU baseline) against the
numpy oracle: host-built tomography matrix bit-identical, pivots identical,
iterates within rounding.  CPU only."""

import numpy as np

from oracle import cpu_baseline as cb
from oracle import hessketch_oracle as ho
from oracle import tomo_oracle as to


def test_host_tomography_matches_oracle():
    A, At, m, n = cb.host_tomography(40, 17, 31, 4)
    K = to.tomography_matrix(40, 17, 31)
    np.testing.assert_array_equal(A[0], K.indptr)
    np.testing.assert_array_equal(A[1], K.indices)
    np.testing.assert_array_equal(A[2], K.data.astype(np.float32))
    Kt = K.T.tocsr()
    np.testing.assert_array_equal(At[0], Kt.indptr)
    np.testing.assert_array_equal(At[1], Kt.indices)
    np.testing.assert_array_equal(At[2], Kt.data.astype(np.float32))


def test_c_port_matches_oracle32():
    from paper_2502_02721_b200.problems import add_noise, random_ellipses

    grid, angles, bins = 48, 30, 69
    A, At, m, n = cb.host_tomography(grid, angles, bins, 4)
    K = to.tomography_matrix(grid, angles, bins)
    x = random_ellipses(grid, 10, 0).ravel()
    b, _ = add_noise(K @ x, 0.01, 1)
    S = cb.sparse_sign(200, m, 8, 3)
    r = cb.run_slslu(A, At, m, n, b, 200, 40, 1e9, 4, S=S)
    ref = ho.hessenberg_solve(ho.csr_operator(K, np.float32), b, square=False, maxiter=40, S2=S, x_true=x)
    t_ref, g_ref = ho.pivots_of(ref.state)
    assert r["done"] == 40
    np.testing.assert_array_equal(r["t"], t_ref)
    np.testing.assert_array_equal(r["g"], g_ref)
    np.testing.assert_allclose(r["sres"], ref.column("sres_norm"), rtol=1e-9)
    assert np.linalg.norm(r["x"] - ref.x) <= 1e-9 * np.linalg.norm(ref.x)


def test_probe_rate_runs_every_step():
    """The reference-arm cost probe times one loop-body iteration at steps
    spread over k = 1..K and averages the interpolated t(k) over every k."""
    grid, angles, bins, K, ell = 48, 30, 69, 40, 200
    A, At, m, n = cb.host_tomography(grid, angles, bins, 4)
    rate, ks, times = cb.probe_rate(A, At, m, n, ell, K, 4, kpoints=5)
    assert ks[0] == 1 and ks[-1] == K and len(ks) == 5
    assert all(t > 0 for t in times)
    assert abs(1.0 / rate - np.mean(np.interp(np.arange(1, K + 1), ks, times))) < 1e-12


def test_c_psf_conv_matches_oracle_stencil():
    """The C stencil used for the full-size config-5 pivot check is the
    oracle's order-specified convolution, bit for bit."""
    from paper_2502_02721_b200.problems import gaussian_psf

    img = np.random.default_rng(1).standard_normal((45, 38)).astype(np.float32)
    for r in (3, 7, 15):
        psf = gaussian_psf(2.0, radius=r)
        np.testing.assert_array_equal(cb.psf_conv(img, psf, 4), to.psf_stencil(img, psf, False, np.float32))


def test_c_scmrh_pivots_match_oracle32():
    from paper_2502_02721_b200.problems import gaussian_psf

    rng = np.random.default_rng(2)
    H, W, K = 40, 36, 25
    psf = gaussian_psf(2.0, radius=7)
    b = rng.standard_normal(H * W)
    t, Hc = cb.scmrh_psf_pivots((H, W), psf, b, K, 4)
    A = ho.Operator(H * W, H * W, lambda v: to.psf_stencil(v.reshape(H, W), psf, False, np.float32).ravel(),
                    lambda v: to.psf_stencil(v.reshape(H, W), psf, True, np.float32).ravel(), np.float32)
    ref = ho.hessenberg_solve(A, b, square=True, maxiter=K, S2=rng.standard_normal((4 * K, H * W)))
    t_ref, _ = ho.pivots_of(ref.state)
    np.testing.assert_array_equal(t, t_ref)
    np.testing.assert_array_equal(Hc, ref.state.H_matrix())
