"""Projected least-squares routines on the device (linops.py:168-229 restated
by hs_projected_ls / the loop's incremental QR): agreement with the normal
equations and the closed-form Tikhonov solution, the rank gate and its
exception, lam = 0 reduction, input validation."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib

    _lib.load()
    return hs


def test_dense_qr_ls_matches_normal_equations(hs):
    rng = np.random.default_rng(1)
    for l, k in ((30, 7), (200, 60), (1200, 300)):
        M = rng.standard_normal((l, k))
        rhs = rng.standard_normal(l)
        y = hs.dense_qr_ls(M, rhs)
        y_ne = np.linalg.solve(M.T @ M, M.T @ rhs)
        np.testing.assert_allclose(y, y_ne, rtol=1e-9, atol=1e-11)
    # square, exactly consistent
    M = rng.standard_normal((9, 9)) + 4 * np.eye(9)
    x = rng.standard_normal(9)
    np.testing.assert_allclose(hs.dense_qr_ls(M, M @ x), x, rtol=1e-12)


def test_dense_qr_ls_rank_gate(hs):
    rng = np.random.default_rng(2)
    M = rng.standard_normal((20, 5))
    M = np.column_stack([M, M[:, 1] + 2 * M[:, 3]])  # dependent sixth column
    with pytest.raises(hs.RankDeficiencyError) as exc:
        hs.dense_qr_ls(M, rng.standard_normal(20))
    assert exc.value.rank == 5
    assert isinstance(exc.value, np.linalg.LinAlgError)
    with pytest.raises(hs.RankDeficiencyError):
        hs.dense_qr_ls(np.zeros((4, 2)), np.ones(4))


def test_stacked_tikhonov_closed_form_and_reduction(hs):
    rng = np.random.default_rng(3)
    M = rng.standard_normal((40, 8))
    N = rng.standard_normal((25, 8))
    rhs = rng.standard_normal(40)
    lam = 0.7
    y = hs.stacked_tikhonov_ls(M, N, rhs, lam)
    y_cf = np.linalg.solve(M.T @ M + lam**2 * N.T @ N, M.T @ rhs)
    np.testing.assert_allclose(y, y_cf, rtol=1e-9, atol=1e-11)
    np.testing.assert_array_equal(hs.stacked_tikhonov_ls(M, N, rhs, 0.0), hs.dense_qr_ls(M, rhs))
    with pytest.raises(ValueError):
        hs.stacked_tikhonov_ls(M, N, rhs, -1.0)
    with pytest.raises(ValueError):
        hs.stacked_tikhonov_ls(M, N[:, :5], rhs, 0.5)


def test_dense_qr_ls_validation(hs):
    with pytest.raises(ValueError):
        hs.dense_qr_ls(np.ones(3), np.ones(3))
    with pytest.raises(ValueError):
        hs.dense_qr_ls(np.ones((2, 3)), np.ones(2))
    with pytest.raises(ValueError):
        hs.dense_qr_ls(np.ones((4, 2)), np.ones(3))
