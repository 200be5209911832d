"""Step-level API on the device (hs_stepper_*, hessenberg.py:160-226, 275-390):
init_square / step_square / init_generalized / step_generalized with the
state resident on the device, checked against the reference's own step
sequences (tests/golden/steps_dense.npz, sampled_unsketched.npz), against the
fused solver loop (same kernels: bit for bit), and for the reference's
observable behaviour (TrivialSolution, RuntimeError after a breakdown,
keep_product(s), counters)."""

import numpy as np
import pytest
import scipy.sparse

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import paper_2502_02721_b200 as hs
    from paper_2502_02721_b200 import _lib

    _lib.load()
    return hs


def test_steps_vs_reference_fixture(hs, golden):
    """Dense step sequences of the reference (square 9 steps; tall / wide until
    breakdown): pivots exact, H / W / bases to the dense-operator tolerance
    (the reference's BLAS row sums vs the device's sequential ones)."""
    g = golden("steps_dense")
    A = hs.LinearOperator.from_matrix(g["sq_M"])
    st = hs.init_square(A, g["sq_b"])
    for _ in range(9):
        hs.step_square(st, A)
    np.testing.assert_array_equal(st.t[: len(st.L_cols)], g["sq_t"])
    np.testing.assert_allclose(st.H_matrix(), g["sq_H"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(st.L_matrix(), g["sq_L"], rtol=1e-10, atol=1e-12)
    for tag in ("tall", "wide"):
        M = g[f"{tag}_M"]
        A = hs.LinearOperator.from_matrix(M)
        st = hs.init_generalized(A, g[f"{tag}_b"])
        for _ in range(min(M.shape) + 2):
            if st.breakdown:
                break
            hs.step_generalized(st, A)
        assert st.breakdown == bool(g[f"{tag}_breakdown"]) and st.k == int(g[f"{tag}_k"])
        np.testing.assert_array_equal(st.t[: len(st.D_cols)], g[f"{tag}_t"])
        np.testing.assert_array_equal(st.g[: len(st.L_cols)], g[f"{tag}_g"])
        np.testing.assert_allclose(st.H_matrix(), g[f"{tag}_H"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(st.W_matrix(), g[f"{tag}_W"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(st.D_matrix(), g[f"{tag}_D"], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(st.L_matrix(), g[f"{tag}_L"], rtol=1e-10, atol=1e-12)
        with pytest.raises(RuntimeError):
            hs.step_generalized(st, A)


def test_sampled_steps_vs_reference(hs, golden):
    """PivotStrategy.sampled(5, seed=13) stepping draws the reference's RNG
    sequence: the pivots of its scmrh run (15 iterations) come out bit for bit."""
    g = golden("sampled_unsketched")
    A = hs.LinearOperator.from_matrix(g["sq_M"])
    st = hs.init_square(A, g["sq_b"], strategy=hs.PivotStrategy.sampled(5, seed=13))
    for _ in range(15):
        hs.step_square(st, A)
    np.testing.assert_array_equal(st.t[: len(g["samp_sq_t"])], g["samp_sq_t"])
    np.testing.assert_allclose(st.H_matrix(), g["samp_sq_H"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_stepping_equals_the_solver_loop(hs, dtype):
    """Same kernels: K steps of init_generalized / step_generalized on the
    tomography operator reproduce the factorization inside slslu bit for bit,
    including a capacity regrowth (capacity 4 < K)."""
    from paper_2502_02721_b200.problems import add_noise, random_ellipses

    grid, angles, bins, K = 32, 20, 45, 14
    vdt = np.float32 if dtype == "float32" else np.float64
    op = hs.TomographyOperator(grid, angles, bins, dtype=vdt)
    x = random_ellipses(grid, 10, 0).ravel()
    b, _ = add_noise(op.matvec(x), 0.01, 1)
    res = hs.slslu(op, b, hs.SolverConfig(maxiter=K, dtype=dtype, sketch_kind="sparse_sign"))
    st = hs.init_generalized(op, b, dtype=dtype, capacity=4)
    for _ in range(K):
        hs.step_generalized(st, op)
    f = res.factorization
    np.testing.assert_array_equal(st.t[: len(st.D_cols)], f.t[: len(st.D_cols)])
    np.testing.assert_array_equal(st.g[: len(st.L_cols)], f.g[: len(st.L_cols)])
    np.testing.assert_array_equal(st.H_matrix(), f.H_matrix())
    np.testing.assert_array_equal(st.W_matrix(), f.W_matrix())
    np.testing.assert_array_equal(st.L_matrix(), f.L_matrix())
    np.testing.assert_array_equal(st.D_matrix(), f.D_matrix())


def test_products_trivial_and_counters(hs):
    rng = np.random.default_rng(5)
    M = scipy.sparse.random(30, 30, density=0.3, random_state=1, format="csr") + scipy.sparse.eye(30) * 3
    A = hs.LinearOperator.from_matrix(M.tocsr())
    b = rng.standard_normal(30)
    Ac = A.with_fresh_counters() if hasattr(A, "with_fresh_counters") else A
    st = hs.init_square(Ac, b)
    hs.step_square(st, Ac, keep_product=True)
    hs.step_square(st, Ac, keep_product=True)
    # the unreduced A l_k (hessenberg.py:206-207): bitwise the CSR row sums of l_2
    np.testing.assert_array_equal(st.last_product, M.tocsr() @ st.L_cols[1])
    assert st.k == 2 and len(st.h_cols) == 2 and len(st.h_cols[1]) == 3
    np.testing.assert_allclose(st.r0, b)
    assert st.beta == b[np.argmax(np.abs(b))]
    if hasattr(Ac, "counters") and Ac.counters is not None:
        assert Ac.counters.matvec_count == 2
    with pytest.raises(hs.TrivialSolution) as exc:
        hs.init_square(A, np.zeros(30))
    np.testing.assert_array_equal(exc.value.x, np.zeros(30))
    with pytest.raises(ValueError):
        hs.init_square(hs.LinearOperator.from_matrix(np.ones((3, 2))), np.ones(3))
    # rectangular: keep_products gives both unreduced products
    R = rng.standard_normal((12, 7))
    Ar = hs.LinearOperator.from_matrix(scipy.sparse.csr_matrix(R))
    sr = hs.init_generalized(Ar, rng.standard_normal(12))
    hs.step_generalized(sr, Ar, keep_products=True)
    np.testing.assert_array_equal(sr.last_data_product, scipy.sparse.csr_matrix(R) @ sr.L_cols[0])
    np.testing.assert_array_equal(sr.last_solution_product, scipy.sparse.csr_matrix(R).T.tocsr() @ sr.D_cols[1])
    # A^T r0 = 0: TrivialSolution from the transposed residual
    with pytest.raises(hs.TrivialSolution):
        hs.init_generalized(hs.LinearOperator.from_matrix(np.array([[1.0], [0.0]])), np.array([0.0, 1.0]))


def test_dump_factorization(hs, tmp_path):
    from paper_2502_02721_b200.linops import load_array

    rng = np.random.default_rng(2)
    R = rng.standard_normal((10, 6))
    A = hs.LinearOperator.from_matrix(R)
    st = hs.init_generalized(A, rng.standard_normal(10))
    for _ in range(3):
        hs.step_generalized(st, A)
    hs.dump_factorization(st, tmp_path, prefix="f_")
    np.testing.assert_allclose(load_array(tmp_path / "f_H.mm"), st.H_matrix())
    np.testing.assert_allclose(load_array(tmp_path / "f_W.mm"), st.W_matrix())
    np.testing.assert_allclose(load_array(tmp_path / "f_pivots_g.mm").ravel(), st.g)


def test_pivot_select_semantics(hs):
    """pivot_select (hessenberg.py:93-115) on the device: signed value of the
    largest |v|, ties toward the smallest row index whatever the listing order,
    all-zero candidates -> value 0.0, sampling draws the reference's subset."""
    full = hs.PivotStrategy.full()
    v = np.array([3.0, -5.0, 2.0])
    assert hs.pivot_select(v, [0, 1, 2], full) == (1, -5.0)
    assert hs.pivot_select(v, [0, 2], full) == (0, 3.0)
    v = np.array([2.0, -2.0, 2.0])
    assert hs.pivot_select(v, [2, 1, 0], full) == (0, 2.0)
    assert hs.pivot_select(v, [2, 1], full) == (1, -2.0)
    assert hs.pivot_select(np.zeros(4), [1, 3], full)[1] == 0.0
    with pytest.raises(ValueError):
        hs.pivot_select(np.ones(3), [], full)
    with pytest.raises(ValueError):
        hs.pivot_select(np.ones(10), list(range(10)), hs.PivotStrategy.sampled(2))
    rng = np.random.default_rng(4)
    w = rng.standard_normal(50)
    adm = np.arange(5, 50)
    strat = hs.PivotStrategy.sampled(7, seed=1)
    got = hs.pivot_select(w, adm, strat, np.random.default_rng(9))
    sub = np.random.default_rng(9).choice(adm, size=7, replace=False)
    i = int(sub[np.argmax(np.abs(w[sub]))])
    assert got == (i, float(w[i]))
    # sample size >= admissible size: the full set
    assert hs.pivot_select(w, adm, hs.PivotStrategy.sampled(45), None) == hs.pivot_select(w, adm, full)
