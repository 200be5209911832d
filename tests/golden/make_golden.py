"""Generate the golden fixtures in tests/golden/*.npz by running the UNMODIFIED
reference package (``/root/reference/pkg/src/hessketch``) in the build
container.  The GPU box has no ``/root/reference``; only the fixtures travel.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each fixture stores the inputs (operator matrix or construction parameters,
b, explicit sketch matrices, config) and the reference outputs (pivot
sequences, H/W, bases, x, per-iteration sres_norm / proj_obj / rel_err /
counters / rank_fallback, termination).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import scipy.sparse

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import hessketch  # noqa: E402
from hessketch import problems, solvers  # noqa: E402
from hessketch.hessenberg import (  # noqa: E402
    GeneralizedHessenbergState,
    PivotStrategy,
    init_generalized,
    init_square,
    step_generalized,
    step_square,
)
from hessketch.linops import LinearOperator  # noqa: E402
from hessketch.sketch import SketchOperator, derive_seed, make_gaussian_sketch  # noqa: E402


def _pack_result(res, prefix=""):
    out = {}
    out[prefix + "x"] = np.asarray(res.x, dtype=np.float64)
    out[prefix + "termination"] = np.array(res.termination)
    recs = res.trace.records
    for name in ("sres_norm", "proj_obj", "rel_err"):
        vals = [getattr(r, name) for r in recs]
        out[prefix + name] = np.array([np.nan if v is None else v for v in vals], dtype=np.float64)
    for name in ("matvecs", "tmatvecs", "dots", "sketches"):
        out[prefix + name] = np.array([getattr(r, name) for r in recs], dtype=np.int64)
    out[prefix + "rank_fallback"] = np.array([r.rank_fallback for r in recs], dtype=bool)
    for name in ("res_norm", "kappa_basis", "kappa_dbar", "eps_embed"):
        if any(getattr(r, name) is not None for r in recs):
            out[prefix + name] = np.array([np.nan if getattr(r, name) is None else getattr(r, name) for r in recs])
    st = res.factorization
    if st is not None:
        out[prefix + "H"] = st.H_matrix()
        if isinstance(st, GeneralizedHessenbergState):
            out[prefix + "t"] = np.asarray(st.t[: len(st.D_cols)], dtype=np.int64)
            out[prefix + "g"] = np.asarray(st.g[: len(st.L_cols)], dtype=np.int64)
            out[prefix + "W"] = st.W_matrix()
            out[prefix + "D"] = np.column_stack(st.D_cols)
            out[prefix + "L"] = np.column_stack(st.L_cols)
        else:
            out[prefix + "t"] = np.asarray(st.t[: len(st.L_cols)], dtype=np.int64)
            out[prefix + "L"] = np.column_stack(st.L_cols)
    return out


def _save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(np.asarray(a).nbytes for a in arrays.values()), "bytes")


def _csr_arrays(M, prefix="A_"):
    M = scipy.sparse.csr_matrix(M)
    return {
        prefix + "indptr": M.indptr.astype(np.int64),
        prefix + "indices": M.indices.astype(np.int32),
        prefix + "data": M.data.astype(np.float64),
        prefix + "shape": np.array(M.shape, dtype=np.int64),
    }


def sparse_sign_entries(ell, m, zeta, seed):
    """A sparse-sign S (zeta +-1/sqrt(zeta) per column) drawn with numpy; the
    reference accepts any ``entries`` supporting ``@`` through ``sketch=``."""
    rng = np.random.default_rng(seed)
    rows = np.concatenate([rng.choice(ell, size=zeta, replace=False) for _ in range(m)])
    cols = np.repeat(np.arange(m), zeta)
    vals = rng.choice([-1.0, 1.0], size=m * zeta) / np.sqrt(zeta)
    return scipy.sparse.csr_matrix((vals, (rows, cols)), shape=(ell, m))


def gen_pivot_and_steps():
    """Hand examples from the reference's own tests plus dense step sequences."""
    rng = np.random.default_rng(17)
    cases = {}
    # square dense steps (no sketch): the pure basis recurrence
    M = rng.standard_normal((12, 12))
    b = rng.standard_normal(12)
    A = LinearOperator.from_matrix(M)
    st = init_square(A, b)
    for _ in range(9):
        step_square(st, A)
    cases.update(sq_M=M, sq_b=b, sq_t=np.asarray(st.t[: len(st.L_cols)]),
                 sq_H=st.H_matrix(), sq_L=np.column_stack(st.L_cols))
    # generalized dense steps, tall and wide
    for tag, shape in (("tall", (14, 9)), ("wide", (7, 11))):
        M = rng.standard_normal(shape)
        b = rng.standard_normal(shape[0])
        A = LinearOperator.from_matrix(M)
        st = init_generalized(A, b)
        for _ in range(min(shape) + 2):
            if st.breakdown:
                break
            step_generalized(st, A)
        cases.update({
            f"{tag}_M": M, f"{tag}_b": b,
            f"{tag}_t": np.asarray(st.t[: len(st.D_cols)]),
            f"{tag}_g": np.asarray(st.g[: len(st.L_cols)]),
            f"{tag}_H": st.H_matrix(), f"{tag}_W": st.W_matrix(),
            f"{tag}_D": np.column_stack(st.D_cols), f"{tag}_L": np.column_stack(st.L_cols),
            f"{tag}_breakdown": np.array(st.breakdown), f"{tag}_k": np.array(st.k),
        })
    _save("steps_dense", **cases)


def gen_scmrh_dense():
    rng = np.random.default_rng(101)
    n = 40
    M = rng.standard_normal((n, n)) + 4.0 * np.eye(n)
    b = rng.standard_normal(n)
    x_true = np.linalg.solve(M, b)
    cfg = solvers.SolverConfig(maxiter=12, seed=5)
    A = LinearOperator.from_matrix(M)
    res = solvers.scmrh(A, b, cfg, x_true=x_true)
    S = make_gaussian_sketch(cfg.effective_sketch_rows(), n, cfg.seed).entries
    out = dict(M=M, b=b, x_true=x_true, S2=S, maxiter=np.array(12), seed=np.array(5))
    out.update(_pack_result(res))
    # same problem, explicit scaled-orthogonal sketch through sketch= (test_solvers.py:287-301 style)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    So = SketchOperator(n, n, seed=0, entries=3.0 * Q)
    res2 = solvers.scmrh(A, b, solvers.SolverConfig(maxiter=8), x_true=x_true, sketch=So)
    out["S2_orth"] = 3.0 * Q
    out.update(_pack_result(res2, "orth_"))
    # x0 given
    x0 = rng.standard_normal(n) * 0.1
    res3 = solvers.scmrh(A, b, solvers.SolverConfig(maxiter=6, seed=2, x0=x0))
    out["x0"] = x0
    out["S2_x0"] = make_gaussian_sketch(70, n, 2).entries
    out.update(_pack_result(res3, "x0_"))
    # Tikhonov (square): S1 from derive_seed
    res4 = solvers.scmrh_tikhonov(A, b, solvers.SolverConfig(maxiter=7, seed=3, lam=0.4))
    out["S2_tik"] = make_gaussian_sketch(80, n, 3).entries
    out["S1_tik"] = make_gaussian_sketch(80, n, derive_seed(3, 1)).entries
    out.update(_pack_result(res4, "tik_"))
    _save("scmrh_dense", **out)


def gen_slslu_dense():
    rng = np.random.default_rng(202)
    m, n = 60, 25
    M = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    x_true = np.linalg.lstsq(M, b, rcond=None)[0]
    A = LinearOperator.from_matrix(M)
    out = dict(M=M, b=b, x_true=x_true)
    cfg = solvers.SolverConfig(maxiter=10, seed=7)
    res = solvers.slslu(A, b, cfg, x_true=x_true)
    out["S2"] = make_gaussian_sketch(110, m, 7).entries
    out.update(_pack_result(res))
    cfgt = solvers.SolverConfig(maxiter=9, seed=3, lam=0.7)
    rest = solvers.slslu_tikhonov(A, b, cfgt, x_true=x_true)
    out["S2_tik"] = make_gaussian_sketch(100, m, 3).entries
    out["S1_tik"] = make_gaussian_sketch(100, n, derive_seed(3, 1)).entries
    out.update(_pack_result(rest, "tik_"))
    # wide system: breakdown on the solution side once L spans R^n
    Mw = rng.standard_normal((8, 5))
    bw = rng.standard_normal(8)
    resw = solvers.slslu(LinearOperator.from_matrix(Mw), bw, solvers.SolverConfig(maxiter=9, seed=1))
    out["Mw"], out["bw"] = Mw, bw
    out["S2_w"] = make_gaussian_sketch(100, 8, 1).entries
    out.update(_pack_result(resw, "w_"))
    # the 2x1 hand example (test_solvers.py:225-233) through the sketched solver
    Mh = np.array([[1.0], [1.0]])
    resh = solvers.slslu(LinearOperator.from_matrix(Mh), np.array([1.0, 3.0]), solvers.SolverConfig(maxiter=1, seed=0))
    out["Mh"] = Mh
    out["S2_h"] = make_gaussian_sketch(20, 2, 0).entries
    out.update(_pack_result(resh, "h_"))
    _save("slslu_dense", **out)


def gen_tomography():
    out = {}
    for grid, angles in ((8, 6), (13, 7), (16, 12)):
        K = problems.tomography_matrix(grid, angles)
        out.update(_csr_arrays(K, prefix=f"tomo{grid}x{angles}_"))
    _save("tomo_matrices", **out)

    # a small sLSLU tomography solve with a sparse-sign S2 through sketch= and
    # a Tikhonov solve with the reference's own Gaussian S1
    prob = problems.make_tomography(16, 12, noise_level=0.01, seed=4)
    K = problems.tomography_matrix(16, 12)
    m = K.shape[0]
    S = sparse_sign_entries(60, m, 8, seed=9)
    sk = SketchOperator(60, m, seed=9, entries=S)
    cfg = solvers.SolverConfig(maxiter=40)
    res = solvers.slslu(prob.operator, prob.b, cfg, x_true=prob.x_true, sketch=sk)
    o = dict(b=prob.b, x_true=prob.x_true, maxiter=np.array(40))
    o.update(_csr_arrays(K))
    o.update(_csr_arrays(S, prefix="S2_"))
    o.update(_pack_result(res))
    cfgt = solvers.SolverConfig(maxiter=30, lam=1e-3, seed=11)
    rest = solvers.slslu(prob.operator, prob.b, cfgt, x_true=prob.x_true, sketch=sk)
    o["S1_tik"] = make_gaussian_sketch(60, K.shape[1], derive_seed(11, 1)).entries
    o.update(_pack_result(rest, "tik_"))
    _save("slslu_tomo16", **o)


def gen_deblur():
    psf = problems.gaussian_psf(1.0, radius=2)
    prob = problems.make_deblur(16, psf, noise_level=0.01, seed=3)
    cfg = solvers.SolverConfig(maxiter=25, seed=6)
    res = solvers.scmrh(prob.operator, prob.b, cfg, x_true=prob.x_true)
    n = 256
    o = dict(psf=psf, b=prob.b, x_true=prob.x_true, size=np.array(16), maxiter=np.array(25))
    o["S2"] = make_gaussian_sketch(260, n, 6).entries
    o.update(_pack_result(res))
    # operator goldens: scipy convolve2d / correlate2d of a fixed image
    img = np.random.default_rng(5).standard_normal((16, 16))
    o["img"] = img
    o["conv"] = prob.operator.forward(img.ravel())
    o["corr"] = prob.operator.transpose(img.ravel())
    _save("scmrh_deblur16", **o)


def gen_edge():
    o = {}
    # identity: lucky breakdown at k = 1 (test_solvers.py:279-284)
    b = np.array([1.0, -2.0, 0.5, 3.0, 1.5])
    res = solvers.scmrh(LinearOperator.identity(5), b, solvers.SolverConfig(maxiter=3, seed=42))
    o["id_b"] = b
    o["id_S2"] = make_gaussian_sketch(40, 5, 42).entries
    o.update(_pack_result(res, "id_"))
    # zero rhs: trivial
    res0 = solvers.slslu(LinearOperator.from_matrix(np.ones((4, 3))), np.zeros(4), solvers.SolverConfig(maxiter=2))
    o["zero_termination"] = np.array(res0.termination)
    o["zero_x"] = res0.x
    # normal equations already hold: A^T b = 0 -> trivial
    res1 = solvers.slslu(LinearOperator.from_matrix(np.array([[1.0], [0.0]])), np.array([0.0, 1.0]), solvers.SolverConfig(maxiter=2))
    o["ne_termination"] = np.array(res1.termination)
    # ties in |r0| resolve to the smallest index
    Mt = np.diag([1.0, 2.0, 3.0, 4.0])
    bt = np.array([2.0, -2.0, 2.0, 1.0])
    rest = solvers.scmrh(LinearOperator.from_matrix(Mt), bt, solvers.SolverConfig(maxiter=3, seed=1))
    o["tie_M"], o["tie_b"] = Mt, bt
    o["tie_S2"] = make_gaussian_sketch(40, 4, 1).entries
    o.update(_pack_result(rest, "tie_"))
    _save("edge_cases", **o)


def gen_sampled_and_unsketched():
    """Sampled pivoting (PivotStrategy.sampled, hessenberg.py:48-124) and the
    unsketched cmrh / lslu (solvers.py:542-559), dense and tomography."""
    o = {}
    rng = np.random.default_rng(303)
    n = 40
    M = rng.standard_normal((n, n)) + 4.0 * np.eye(n)
    b = rng.standard_normal(n)
    x_true = np.linalg.solve(M, b)
    A = LinearOperator.from_matrix(M)
    o.update(sq_M=M, sq_b=b, sq_x_true=x_true)
    # sampled scmrh (Gaussian S2 from cfg.seed)
    cfg = solvers.SolverConfig(maxiter=15, seed=5, pivot=PivotStrategy.sampled(5, seed=13))
    o["samp_sq_S2"] = make_gaussian_sketch(cfg.effective_sketch_rows(), n, 5).entries
    o.update(_pack_result(solvers.scmrh(A, b, cfg, x_true=x_true), "samp_sq_"))
    # unsketched cmrh, lam = 0 and lam > 0
    o.update(_pack_result(solvers.cmrh(A, b, solvers.SolverConfig(maxiter=15), x_true=x_true), "cmrh_"))
    o.update(_pack_result(solvers.cmrh(A, b, solvers.SolverConfig(maxiter=12, lam=0.3), x_true=x_true), "cmrh_tik_"))
    # sampled cmrh on a banded operator with a sparse right-hand side: the
    # sampled subsets miss every nonzero early on (full-scan fallback)
    Mb = np.diag(np.full(n, 3.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, 0.5), -1)
    bb = np.zeros(n)
    bb[7] = 1.0
    o.update(band_M=Mb, band_b=bb)
    o.update(_pack_result(
        solvers.cmrh(LinearOperator.from_matrix(Mb), bb, solvers.SolverConfig(maxiter=10, pivot=PivotStrategy.sampled(3, seed=4))),
        "band_"))
    # rectangular: sampled slslu, unsketched lslu (lam 0 / > 0), sampled lslu
    rng = np.random.default_rng(404)
    m, nn = 60, 25
    Mr = rng.standard_normal((m, nn))
    br = rng.standard_normal(m)
    xr = np.linalg.lstsq(Mr, br, rcond=None)[0]
    Ar = LinearOperator.from_matrix(Mr)
    o.update(re_M=Mr, re_b=br, re_x_true=xr)
    cfg = solvers.SolverConfig(maxiter=12, seed=7, pivot=PivotStrategy.sampled(4, seed=2))
    o["samp_re_S2"] = make_gaussian_sketch(cfg.effective_sketch_rows(), m, 7).entries
    o.update(_pack_result(solvers.slslu(Ar, br, cfg, x_true=xr), "samp_re_"))
    o.update(_pack_result(solvers.lslu(Ar, br, solvers.SolverConfig(maxiter=12), x_true=xr), "lslu_"))
    o.update(_pack_result(solvers.lslu(Ar, br, solvers.SolverConfig(maxiter=10, lam=0.5), x_true=xr), "lslu_tik_"))
    o.update(_pack_result(
        solvers.lslu(Ar, br, solvers.SolverConfig(maxiter=10, pivot=PivotStrategy.sampled(6, seed=1)), x_true=xr),
        "lslu_samp_"))
    # tomography 16^2 x 12 angles: sampled sLSLU through sketch= (sparse-sign), unsketched LSLU
    prob = problems.make_tomography(16, 12, noise_level=0.01, seed=4)
    K = problems.tomography_matrix(16, 12)
    S = sparse_sign_entries(60, K.shape[0], 8, seed=9)
    sk = SketchOperator(60, K.shape[0], seed=9, entries=S)
    o.update(tomo_b=prob.b, tomo_x_true=prob.x_true)
    o.update(_csr_arrays(S, prefix="tomo_S2_"))
    o.update(_pack_result(
        solvers.slslu(prob.operator, prob.b, solvers.SolverConfig(maxiter=30, pivot=PivotStrategy.sampled(25, seed=8)),
                      x_true=prob.x_true, sketch=sk), "tomo_samp_"))
    o.update(_pack_result(solvers.lslu(prob.operator, prob.b, solvers.SolverConfig(maxiter=30), x_true=prob.x_true),
                          "tomo_lslu_"))
    _save("sampled_unsketched", **o)


def gen_exchange():
    """Phantoms, motion PSFs, PGM bytes / error messages and MatrixMarket text
    from the reference (problems.py:152-233, 377-473; linops.py:249-282)."""
    import tempfile

    import scipy.io
    from hessketch import linops

    o = dict(deblur37=problems.deblur_phantom(37), tomo29=problems.tomography_phantom(29),
             deblur8=problems.deblur_phantom(8))
    for i, (length, ang) in enumerate(((7, 30.0), (5, 90.0), (1, 0.0), (9.5, -20.0), (4, 45.0))):
        o[f"motion{i}"] = problems.motion_psf(length, ang)
        o[f"motion{i}_args"] = np.array([length, ang])
    rng = np.random.default_rng(12)
    px = rng.random((5, 7))
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "a.pgm")
        problems.write_image(problems.Image(width=7, height=5, pixels=px), path)
        o["pgm_pixels"] = px
        o["pgm_bytes"] = np.frombuffer(open(path, "rb").read(), dtype=np.uint8)
        good8 = b"P5 # comment\n3 2\n255\n" + bytes([0, 10, 20, 255, 128, 1])
        bad = [b"P6\n1 1\n255\n\x00", b"P5\n0 1\n255\n\x00", b"P5\n2 2\n70000\n" + b"\x00" * 8,
               b"P5\n2 2\n255", b"P5\n2 2\n255\n\x00", b"P5\nx 2\n255\n\x00", b"P5\n2"]
        msgs = []
        for i, blob in enumerate([good8] + bad):
            fp = os.path.join(d, f"b{i}.pgm")
            open(fp, "wb").write(blob)
            try:
                img = problems.read_image(fp)
                msgs.append("ok")
                o["pgm8_pixels"] = img.pixels
            except problems.ImageFormatError as e:
                msgs.append(str(e))
            o[f"pgm_case{i}"] = np.frombuffer(blob, dtype=np.uint8)
        o["pgm_msgs"] = np.array(msgs)
        M = rng.standard_normal((4, 3))
        v = rng.standard_normal(5)
        for name, arr in (("mtx_mat", M), ("mtx_vec", v)):
            fp = os.path.join(d, name + ".mtx")
            linops.save_array(fp, arr)
            o[name] = arr
            o[name + "_bytes"] = np.frombuffer(open(fp, "rb").read(), dtype=np.uint8)
        S = scipy.sparse.random(6, 5, density=0.4, random_state=3, format="csr")
        fp = os.path.join(d, "coo.mtx")
        with open(fp, "wb") as fh:
            scipy.io.mmwrite(fh, S)
        o["coo_bytes"] = np.frombuffer(open(fp, "rb").read(), dtype=np.uint8)
        o["coo_dense"] = S.toarray()
    o["cond"] = np.array([linops.spectral_condition_number(np.array([[3.0, 0.0], [0.0, 0.5]])),
                          linops.spectral_condition_number(np.diag([1.0, 1e-301]))])
    _save("exchange", **o)


def gen_krylov():
    """The comparison solvers gmres / lsqr (solvers.py:256-403), with
    diagnostics (res_norm), damping, x0, lucky breakdown and exhaustion."""
    o = {}
    rng = np.random.default_rng(505)
    n = 40
    M = rng.standard_normal((n, n)) + 4.0 * np.eye(n)
    b = rng.standard_normal(n)
    xt = np.linalg.solve(M, b)
    A = LinearOperator.from_matrix(M)
    o.update(sq_M=M, sq_b=b, sq_x_true=xt)
    diag = solvers.SolverConfig(maxiter=15, compute_diagnostics=True)
    o.update(_pack_result(solvers.gmres(A, b, diag, x_true=xt), "gm_"))
    o.update(_pack_result(solvers.gmres(A, b, solvers.SolverConfig(maxiter=12, lam=0.3), x_true=xt), "gm_tik_"))
    x0 = rng.standard_normal(n) * 0.1
    o["x0"] = x0
    o.update(_pack_result(solvers.gmres(A, b, solvers.SolverConfig(maxiter=8, x0=x0, compute_diagnostics=True)), "gm_x0_"))
    o.update(_pack_result(solvers.gmres(LinearOperator.identity(3), np.array([3.0, -5.0, 2.0])), "gm_id_"))
    rng = np.random.default_rng(606)
    m, nn = 60, 25
    Mr = rng.standard_normal((m, nn))
    br = rng.standard_normal(m)
    xr = np.linalg.lstsq(Mr, br, rcond=None)[0]
    Ar = LinearOperator.from_matrix(Mr)
    o.update(re_M=Mr, re_b=br, re_x_true=xr)
    o.update(_pack_result(solvers.lsqr(Ar, br, solvers.SolverConfig(maxiter=15, compute_diagnostics=True), x_true=xr), "ls_"))
    o.update(_pack_result(solvers.lsqr(Ar, br, solvers.SolverConfig(maxiter=10, lam=0.5), x_true=xr), "ls_tik_"))
    x0r = rng.standard_normal(nn) * 0.1
    o["x0r"] = x0r
    o.update(_pack_result(solvers.lsqr(Ar, br, solvers.SolverConfig(maxiter=8, x0=x0r)), "ls_x0_"))
    Mw = rng.standard_normal((8, 3))
    bw = rng.standard_normal(8)
    o.update(w_M=Mw, w_b=bw)
    o.update(_pack_result(solvers.lsqr(LinearOperator.from_matrix(Mw), bw, solvers.SolverConfig(maxiter=6)), "ls_w_"))
    prob = problems.make_tomography(16, 12, noise_level=0.01, seed=4)
    o.update(_pack_result(solvers.lsqr(prob.operator, prob.b, solvers.SolverConfig(maxiter=30, compute_diagnostics=True),
                                       x_true=prob.x_true), "ls_tomo_"))
    _save("krylov", **o)


def gen_diagnostics():
    """compute_diagnostics on the Hessenberg solvers (solvers.py:523-532):
    res_norm, kappa_basis, kappa_dbar (lam > 0), eps_embed."""
    o = {}
    rng = np.random.default_rng(707)
    n = 30
    M = rng.standard_normal((n, n)) + 4.0 * np.eye(n)
    b = rng.standard_normal(n)
    A = LinearOperator.from_matrix(M)
    o.update(sq_M=M, sq_b=b)
    o["sq_S2"] = make_gaussian_sketch(130, n, 3).entries
    o.update(_pack_result(solvers.scmrh(A, b, solvers.SolverConfig(maxiter=12, seed=3, compute_diagnostics=True)), "sc_"))
    o["sqt_S2"] = make_gaussian_sketch(130, n, 4).entries
    o["sqt_S1"] = make_gaussian_sketch(130, n, derive_seed(4, 1)).entries
    o.update(_pack_result(solvers.scmrh_tikhonov(A, b, solvers.SolverConfig(maxiter=10, seed=4, lam=0.2,
                                                                             compute_diagnostics=True)), "sct_"))
    o.update(_pack_result(solvers.cmrh(A, b, solvers.SolverConfig(maxiter=12, compute_diagnostics=True)), "cm_"))
    m, nn = 50, 20
    Mr = rng.standard_normal((m, nn))
    br = rng.standard_normal(m)
    Ar = LinearOperator.from_matrix(Mr)
    o.update(re_M=Mr, re_b=br)
    o["re_S2"] = make_gaussian_sketch(120, m, 5).entries
    o["re_S1"] = make_gaussian_sketch(120, nn, derive_seed(5, 1)).entries
    o.update(_pack_result(solvers.slslu_tikhonov(Ar, br, solvers.SolverConfig(maxiter=11, seed=5, lam=0.3,
                                                                               compute_diagnostics=True)), "sl_"))
    o.update(_pack_result(solvers.lslu(Ar, br, solvers.SolverConfig(maxiter=11, compute_diagnostics=True)), "ll_"))
    _save("diagnostics", **o)


def gen_rank_fallback():
    """Low-rank operators: the sketched projected system becomes rank deficient
    (pivoted-QR gate, linops.py:197-203) and the reference takes the lstsq
    minimum-norm fallback from then on (solvers.py:204-218)."""
    rng = np.random.default_rng(0)
    o = {}
    n = 20
    M = rng.standard_normal((n, 3)) @ rng.standard_normal((3, n))
    b = rng.standard_normal(n)
    xt = rng.standard_normal(n)
    # stored as CSR: past the operator's rank the remainders are rounding noise,
    # so the pivots match only under the sequential csr_matvec order the
    # device reproduces bit for bit
    A = LinearOperator.from_matrix(scipy.sparse.csr_matrix(M))
    o.update(sq_M=M, sq_b=b, sq_xt=xt)
    o.update(_pack_result(solvers.scmrh(A, b, solvers.SolverConfig(maxiter=8, sketch_rows=40, seed=1), x_true=xt),
                          "sq_"))
    o.update(_pack_result(solvers.cmrh(A, b, solvers.SolverConfig(maxiter=8), x_true=xt), "cm_"))
    m = 30
    Mr = rng.standard_normal((m, 4)) @ rng.standard_normal((4, n))
    br = rng.standard_normal(m)
    Ar = LinearOperator.from_matrix(scipy.sparse.csr_matrix(Mr))
    o.update(re_M=Mr, re_b=br)
    o.update(_pack_result(solvers.slslu(Ar, br, solvers.SolverConfig(maxiter=9, sketch_rows=40, seed=3), x_true=xt),
                          "re_"))
    o.update(_pack_result(solvers.lslu(Ar, br, solvers.SolverConfig(maxiter=9), x_true=xt), "ll_"))
    for p in ("sq_", "cm_", "re_", "ll_"):
        print(p, "rank_fallback", o[p + "rank_fallback"].astype(int), o[p + "termination"])
    _save("rank_fallback", **o)


def gen_printed_f():
    """slslu_tikhonov(printed_f_columns=True): penalty columns from the
    unreduced A^T d_{k+1} (solvers.py:460-461, 488-490, 594-605)."""
    rng = np.random.default_rng(11)
    M = rng.standard_normal((31, 24))
    b = rng.standard_normal(31)
    xt = rng.standard_normal(24)
    A = LinearOperator.from_matrix(M)
    o = dict(M=M, b=b, xt=xt)
    cfg = solvers.SolverConfig(maxiter=8, seed=6, lam=0.5)
    o.update(_pack_result(solvers.slslu_tikhonov(A, b, cfg, x_true=xt, printed_f_columns=True), "pr_"))
    o.update(_pack_result(solvers.slslu_tikhonov(A, b, cfg, x_true=xt), "df_"))
    _save("printed_f", **o)


if __name__ == "__main__":
    print("reference hessketch", hessketch.__version__)
    if len(sys.argv) > 1:  # regenerate selected fixtures only: make_golden.py gen_rank_fallback ...
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    gen_pivot_and_steps()
    gen_scmrh_dense()
    gen_slslu_dense()
    gen_tomography()
    gen_deblur()
    gen_edge()
    gen_sampled_and_unsketched()
    gen_exchange()
    gen_krylov()
    gen_diagnostics()
    gen_rank_fallback()
    gen_printed_f()
