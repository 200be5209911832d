"""Drop-in Hessenberg solvers: the sketched ``scmrh``, ``slslu``,
``scmrh_tikhonov``, ``slslu_tikhonov`` and the unsketched ``cmrh``, ``lslu``
with the reference's signatures and result types (solvers.py:88-160,
542-605), running the whole iteration loop on the B200 through one C-ABI call
(``hs_solve``, restating ``_hessenberg_solve``, solvers.py:410-539).  Full and
sampled pivoting (``PivotStrategy.sampled``, hessenberg.py:48-124) both run on
the device; for the sampled strategy the host draws the positions with the
reference's ``default_rng(seed).choice`` sequence before the loop.

Device knobs added to :class:`SolverConfig` (defaults reproduce the reference):

* ``dtype``        -- "float64" (reference arithmetic) or "float32"
* ``basis_dtype``  -- storage of the Krylov bases: None (= dtype), "float32"
                      or "bfloat16" (with dtype float32)
* ``sketch_kind``  -- how S2 (and S1 when lam > 0) are realised when no
                      ``sketch=`` is passed: "pcg64" (the reference's host
                      draw, sketch.py:43-53, uploaded once; default),
                      "gaussian" (device Philox, never stored) or
                      "sparse_sign" (``sketch_zeta`` nonzeros per column)
* ``record_rel_err`` -- compute rel_err at every iteration (default True when
                      x_true is given, as the reference does)

The reference's comparison solvers ``gmres`` / ``lsqr`` (solvers.py:256-403)
also run on the device (``hs_solve_krylov``).

``compute_diagnostics=True`` computes, on the device, every iteration: the
exact residual ``res_norm`` = |b - A x_k| (solvers.py:247-250, 523-525), the
basis condition number ``kappa_basis`` and, with lam > 0, ``kappa_dbar``
(``_union_condition``, solvers.py:228-233, 526-530; incremental QR of the
bases + Jacobi SVD of the small R factors), and the measured embedding
distortion ``eps_embed`` of S2 on span[A l_1..A l_k, r0] (sketch.py:91-112;
not for ``sketch_basis=True``).  The loop is serialised while diagnostics are
on.  ``slslu_tikhonov(..., printed_f_columns=True)`` runs the reference's
comparison variant (penalty columns from the unreduced A^T d_{k+1},
solvers.py:460-461, 488-490) on the device too.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .hessenberg import DeviceFactorization, PivotStrategy
from .linops import to_device_operator
from .sketch import (
    GaussianSketch,
    SparseSignSketch,
    derive_seed,
    device_sketch,
    make_gaussian_sketch,
)

__all__ = [
    "CSV_COLUMNS",
    "SolverConfig",
    "TraceRecord",
    "SolverTrace",
    "SolveResult",
    "trace_to_csv",
    "scmrh",
    "slslu",
    "scmrh_tikhonov",
    "slslu_tikhonov",
    "cmrh",
    "lslu",
    "gmres",
    "lsqr",
    "SOLVERS",
]

CSV_COLUMNS = [
    "iter", "res_norm", "sres_norm", "proj_obj", "rel_err", "kappa_basis", "kappa_dbar",
    "eps_embed", "matvecs", "tmatvecs", "dots", "sketches", "wall_ms",
]


@dataclass
class SolverConfig:
    """solvers.py:88-116 plus device knobs (module docstring)."""

    maxiter: int = 30
    pivot: PivotStrategy = field(default_factory=PivotStrategy.full)
    sketch_rows: int = None
    lam: float = 0.0
    seed: int = 0
    x0: np.ndarray = None
    compute_diagnostics: bool = False
    dtype: str = "float64"
    basis_dtype: str = None
    sketch_kind: str = "pcg64"
    sketch_zeta: int = 8
    record_rel_err: bool = True

    def __post_init__(self):
        if self.maxiter < 1:
            raise ValueError("maxiter must be positive")
        if self.lam < 0:
            raise ValueError("lam must be nonnegative")
        if self.sketch_rows is not None and self.sketch_rows < 1:
            raise ValueError("sketch_rows must be positive")
        if self.dtype not in ("float64", "float32"):
            raise ValueError("dtype must be 'float64' or 'float32'")
        if self.basis_dtype not in (None, "float64", "float32", "bfloat16"):
            raise ValueError("basis_dtype must be None, 'float64', 'float32' or 'bfloat16'")
        if self.sketch_kind not in ("pcg64", "gaussian", "sparse_sign"):
            raise ValueError("sketch_kind must be 'pcg64', 'gaussian' or 'sparse_sign'")

    def effective_sketch_rows(self):
        if self.sketch_rows is None:
            return 10 * (self.maxiter + 1)
        return self.sketch_rows


@dataclass
class TraceRecord:
    """solvers.py:119-141."""

    iteration: int
    res_norm: float = None
    sres_norm: float = None
    proj_obj: float = None
    rel_err: float = None
    kappa_basis: float = None
    kappa_dbar: float = None
    eps_embed: float = None
    matvecs: int = 0
    tmatvecs: int = 0
    dots: int = 0
    sketches: int = 0
    wall_ms: float = None
    rank_fallback: bool = False


@dataclass
class SolverTrace:
    records: list = field(default_factory=list)

    def column(self, name):
        return [getattr(r, name) for r in self.records]

    def final(self):
        return self.records[-1] if self.records else None


@dataclass
class SolveResult:
    x: np.ndarray
    trace: SolverTrace
    termination: str  # maxiter | breakdown | trivial
    factorization: object = None
    loop_ms: float = None  # device time of the iteration loop (CUDA events)


def _cell(value):
    if value is None:
        return ""
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    return repr(float(value))


def trace_to_csv(trace, target, include_timing=False):
    """solvers.py:171-201 (fixed column order, wall_ms only on request)."""
    lines = [",".join(CSV_COLUMNS)]
    for r in trace.records:
        cells = [
            str(r.iteration), _cell(r.res_norm), _cell(r.sres_norm), _cell(r.proj_obj), _cell(r.rel_err),
            _cell(r.kappa_basis), _cell(r.kappa_dbar), _cell(r.eps_embed), str(r.matvecs), str(r.tmatvecs),
            str(r.dots), str(r.sketches), _cell(r.wall_ms) if include_timing else "",
        ]
        lines.append(",".join(cells))
    content = "\n".join(lines) + "\n"
    if hasattr(target, "write"):
        target.write(content)
    else:
        with open(target, "w", newline="") as fh:
            fh.write(content)


# ---------------------------------------------------------------------------


class _NativeResult:
    """Owns an hs_result handle and its host copies."""

    def __init__(self, handle, rows, cols, ell):
        lib = _lib.load()
        self.handle = handle
        v = [_lib.c_i32() for _ in range(6)]
        _lib.check(lib.hs_result_info(handle, *[ctypes.byref(x) for x in v]))
        nrec, term, k, bds, nbd, nbs = (x.value for x in v)
        self.info = {"n_records": nrec, "termination": _lib.TERMINATIONS[term], "k": k, "bd_side": bds,
                     "n_basis_data": nbd, "n_basis_sol": nbs}
        self.x = np.empty(cols)
        _lib.check(lib.hs_result_x(handle, _lib.ptr(self.x)))
        n = max(nrec, 1)
        self.resnorm = np.full(n, np.nan)
        self.kappa_basis, self.kappa_dbar, self.eps_embed = (np.full(n, np.nan) for _ in range(3))
        if nrec:
            _lib.check(lib.hs_result_resnorm(handle, _lib.ptr(self.resnorm)))
            _lib.check(lib.hs_result_diagnostics(handle, _lib.ptr(self.kappa_basis), _lib.ptr(self.kappa_dbar),
                                                 _lib.ptr(self.eps_embed)))
        self.sres, self.proj, self.relerr, self.wall = (np.empty(n) for _ in range(4))
        self.rankfb = np.empty(n, dtype=np.int32)
        self.matvecs, self.tmatvecs, self.dots, self.sketches = (np.empty(n, dtype=np.int64) for _ in range(4))
        _lib.check(lib.hs_result_trace(handle, *(_lib.ptr(a) for a in (
            self.sres, self.proj, self.relerr, self.rankfb, self.matvecs, self.tmatvecs, self.dots, self.sketches,
            self.wall))))
        self.pivots_t = np.empty(max(nbd, 1), dtype=np.int64)[:nbd]
        self.pivots_g = np.empty(max(nbs, 1), dtype=np.int64)[:nbs]
        if nrec:
            tbuf = np.empty(max(nbd, nbs, 1), dtype=np.int64)
            gbuf = np.empty(max(nbd, nbs, 1), dtype=np.int64)
            _lib.check(lib.hs_result_pivots(handle, _lib.ptr(tbuf), _lib.ptr(gbuf)))
            self.pivots_t = tbuf[:nbd].copy()
            self.pivots_g = gbuf[:nbs].copy()
            Hc = np.empty((k, k + 1))  # column-major (k+1) x k
            Wc = np.empty((max(nbd, 1), max(nbd, 1)))
            _lib.check(lib.hs_result_hessenberg(handle, _lib.ptr(Hc), _lib.ptr(Wc)))
            self.H = np.ascontiguousarray(Hc.T)
            self.W = np.ascontiguousarray(Wc[:nbd, :nbd].T)
            Zc = np.empty((k, ell))
            self.sr0 = np.empty(ell)
            self.y = np.empty(k)
            _lib.check(lib.hs_result_projected(handle, _lib.ptr(Zc), _lib.ptr(self.sr0), _lib.ptr(self.y)))
            self.Z = np.ascontiguousarray(Zc.T)
        ms = _lib.c_dbl()
        _lib.check(lib.hs_result_loop_ms(handle, ctypes.byref(ms)))
        self.loop_ms = ms.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None:
            try:
                _lib.load().hs_result_destroy(h)
            except Exception:
                pass
            self.handle = None


def _opt(v):
    """NaN (not computed) -> None, as the reference's optional trace fields."""
    v = float(v)
    return None if np.isnan(v) else v


# Default sketches realised on the device, reused across solves with the same
# (kind, shape, seed, context): the reference draws S again on every call
# (solvers.py:452-459) with the same bits, so a repeated solve may reuse the
# uploaded matrix.  The PCG64 draw is host work (~5 ms for config 1's 400 x 1024)
# that would otherwise dominate a short solve's end-to-end time.  Bounded: a
# few entries of at most 256 MB of device memory each.
_SKETCH_CACHE = {}
_SKETCH_CACHE_MAX, _SKETCH_CACHE_BYTES = 4, 256 << 20


def _default_sketch(cfg, ell, in_rows, seed):
    from . import _lib

    ctx = _lib.context()
    # only sketches of the process-wide contexts are kept (in-process rank
    # contexts are closed by their owner)
    cacheable = _lib._ctx.get(ctx.device) is ctx
    key = (cfg.sketch_kind, int(ell), int(in_rows), int(seed), cfg.sketch_zeta, ctx.device)
    hit = _SKETCH_CACHE.get(key) if cacheable else None
    if hit is not None:
        return hit
    if cfg.sketch_kind == "pcg64":
        sk = device_sketch(make_gaussian_sketch(ell, in_rows, seed))
    elif cfg.sketch_kind == "gaussian":
        sk = GaussianSketch(ell, in_rows, seed)
    else:
        sk = SparseSignSketch(ell, in_rows, seed, cfg.sketch_zeta)
    nbytes = {"pcg64": 8 * ell * in_rows, "sparse_sign": 3 * in_rows * cfg.sketch_zeta}.get(cfg.sketch_kind, 0)
    if cacheable and nbytes <= _SKETCH_CACHE_BYTES:
        if len(_SKETCH_CACHE) >= _SKETCH_CACHE_MAX:
            _SKETCH_CACHE.pop(next(iter(_SKETCH_CACHE)))
        _SKETCH_CACHE[key] = sk
    return sk


def pivot_positions(strategy, maxiter, rows, cols, square):
    """The draws of the sampled strategy in the reference's order
    (hessenberg.py:171-173, 289-301, 214, 352, 376): one slot per selection,
    ``default_rng(seed).choice(pop, s, replace=False)`` whenever s < pop.
    ``rng.choice(t[k:], s)`` equals ``t[k:][rng.choice(pop, s)]`` with the
    same generator state afterwards, so positions suffice; the device maps
    them through its copy of the swap-ordered permutation."""
    s = int(strategy.sample_size)
    rng = np.random.default_rng(strategy.seed)
    if square:
        pops = [rows] + [rows - k for k in range(1, maxiter + 1)]
    else:
        pops = [rows, cols]
        for k in range(1, maxiter + 1):
            pops += [rows - k, cols - k]
    out = np.full((len(pops), s), -1, dtype=np.int64)
    for slot, pop in enumerate(pops):
        if pop > 0 and s < pop:
            out[slot] = rng.choice(pop, size=s, replace=False)
    return out


def _hessenberg_solve(A, b, cfg, x_true, square, sketch_basis, sketch=None, S1=None, sketched=True,
                      printed_f=False):
    """solvers.py:410-539 on the device (sketched or unsketched branch)."""
    cfg = cfg or SolverConfig()
    if square and not A.is_square:
        raise ValueError("this solver needs a square operator")
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.shape != (A.rows,):
        raise ValueError(f"b must have length {A.rows}, got shape {b.shape}")
    x0 = None if cfg.x0 is None else np.ascontiguousarray(cfg.x0, dtype=np.float64)
    if x0 is None and not np.any(b):
        # hessenberg.py:171-173 / 290-291: zero initial residual, no iteration
        return SolveResult(x=np.zeros(A.cols), trace=SolverTrace(), termination="trivial")
    dev = to_device_operator(A)
    positions = None
    if cfg.pivot.kind == "sampled":
        positions = pivot_positions(cfg.pivot, cfg.maxiter, A.rows, A.cols, square)
    if not sketched:
        ell = cfg.maxiter + 1
        S2 = S1 = None
    elif sketch is not None:
        if sketch.in_rows != A.rows:
            raise ValueError(
                f"sketch expects vectors of length {sketch.in_rows}, operator produces length {A.rows}"
            )
        ell = sketch.out_rows
    else:
        ell = cfg.effective_sketch_rows()
    if sketched:
        if ell < cfg.maxiter + 1:
            raise ValueError(
                f"sketch_rows={ell} cannot embed a {cfg.maxiter}-dimensional projected problem; "
                "need at least maxiter+1 rows"
            )
        S2 = device_sketch(sketch) if sketch is not None else _default_sketch(cfg, ell, A.rows, cfg.seed)
        if cfg.lam > 0.0:
            S1 = device_sketch(S1) if S1 is not None else _default_sketch(cfg, ell, A.cols, derive_seed(cfg.seed, 1))
        else:
            S1 = None
    if x_true is not None:
        x_true = np.ascontiguousarray(x_true, dtype=np.float64)
    basis_dtype = cfg.basis_dtype or cfg.dtype
    if cfg.dtype == "float64" and basis_dtype != "float64":
        raise ValueError("float64 work needs float64 basis storage")
    hc = _lib.HsConfig(
        maxiter=cfg.maxiter, square=1 if square else 0, sketch_basis=1 if sketch_basis else 0,
        work_dtype=_lib.DTYPE_CODES[cfg.dtype], basis_dtype=_lib.DTYPE_CODES[basis_dtype],
        record_x=1 if (x_true is not None and cfg.record_rel_err) else 0, lam=float(cfg.lam),
        sketched=1 if sketched else 0, pivot_sample=0 if positions is None else int(cfg.pivot.sample_size),
        pivot_positions=None if positions is None else positions.ctypes.data,
        diagnostics=1 if cfg.compute_diagnostics else 0,
        printed_f=1 if printed_f else 0,
    )
    h = _lib.c_vp()
    _lib.check(_lib.load().hs_solve(dev.ctx.handle, dev.handle, ctypes.byref(hc),
                                    S2.handle if S2 is not None else None,
                                    S1.handle if S1 is not None else None, _lib.ptr(b), _lib.ptr(x0),
                                    _lib.ptr(x_true), ctypes.byref(h)))
    nr = _NativeResult(h, A.rows, A.cols, ell)
    term = nr.info["termination"]
    if term == "trivial":
        return SolveResult(x=nr.x, trace=SolverTrace(), termination="trivial")
    trace = SolverTrace()
    for i in range(nr.info["n_records"]):
        rel = float(nr.relerr[i])
        trace.records.append(TraceRecord(
            iteration=i + 1,
            sres_norm=float(nr.sres[i]) if sketched else None,
            proj_obj=float(nr.proj[i]),
            rel_err=None if (x_true is None or np.isnan(rel)) else rel,
            res_norm=float(nr.resnorm[i]) if cfg.compute_diagnostics else None,
            kappa_basis=_opt(nr.kappa_basis[i]) if cfg.compute_diagnostics else None,
            kappa_dbar=_opt(nr.kappa_dbar[i]) if cfg.compute_diagnostics else None,
            eps_embed=_opt(nr.eps_embed[i]) if cfg.compute_diagnostics else None,
            matvecs=int(nr.matvecs[i]), tmatvecs=int(nr.tmatvecs[i]), dots=int(nr.dots[i]),
            sketches=int(nr.sketches[i]), wall_ms=float(nr.wall[i]), rank_fallback=bool(nr.rankfb[i]),
        ))
    # a row-sharded solve keeps this rank's rows of the bases (hs_op_shard_info)
    loc = [_lib.c_i64() for _ in range(6)]
    _lib.check(_lib.load().hs_op_shard_info(dev.handle, *[ctypes.byref(v) for v in loc]))
    fact = DeviceFactorization(nr, square, A.rows, A.cols, basis_rows=(loc[1].value, loc[4].value))
    return SolveResult(x=nr.x, trace=trace, termination=term, factorization=fact, loop_ms=nr.loop_ms)


def scmrh(A, b, cfg=None, x_true=None, *, sketch_basis=False, sketch=None):
    """Sketched projected minimal residual on the square Hessenberg basis
    (solvers.py:562-574)."""
    return _hessenberg_solve(A, b, cfg, x_true, True, sketch_basis, sketch)


def slslu(A, b, cfg=None, x_true=None, *, sketch_basis=False, sketch=None):
    """Sketched projected least squares on the generalized bases (solvers.py:577-581)."""
    return _hessenberg_solve(A, b, cfg, x_true, False, sketch_basis, sketch)


def scmrh_tikhonov(A, b, cfg=None, x_true=None):
    """scmrh with the sketched penalty lam^2 |S1 L_k y|^2 (solvers.py:584-591)."""
    return _hessenberg_solve(A, b, cfg, x_true, True, False)


def slslu_tikhonov(A, b, cfg=None, x_true=None, *, printed_f_columns=False):
    """slslu with the sketched penalty (solvers.py:594-605)."""
    return _hessenberg_solve(A, b, cfg, x_true, False, False, printed_f=bool(printed_f_columns))


def _krylov_solve(A, b, cfg, x_true, method):
    """gmres / lsqr (solvers.py:256-403) on the device through ``hs_solve_krylov``."""
    cfg = cfg or SolverConfig()
    b = np.ascontiguousarray(b, dtype=np.float64)
    if b.shape != (A.rows,):
        raise ValueError(f"b must have length {A.rows}, got shape {b.shape}")
    x0 = None if cfg.x0 is None else np.ascontiguousarray(cfg.x0, dtype=np.float64)
    dev = to_device_operator(A)
    if x_true is not None:
        x_true = np.ascontiguousarray(x_true, dtype=np.float64)
    hc = _lib.HsConfig(maxiter=cfg.maxiter, square=1 if method == 0 else 0, sketch_basis=0,
                       work_dtype=_lib.DTYPE_CODES[cfg.dtype], basis_dtype=_lib.DTYPE_CODES[cfg.dtype],
                       record_x=1 if x_true is not None else 0, lam=float(cfg.lam), sketched=0, pivot_sample=0,
                       pivot_positions=None, diagnostics=1 if cfg.compute_diagnostics else 0)
    h = _lib.c_vp()
    _lib.check(_lib.load().hs_solve_krylov(dev.ctx.handle, dev.handle, ctypes.byref(hc), method, _lib.ptr(b),
                                           _lib.ptr(x0), _lib.ptr(x_true), ctypes.byref(h)))
    nr = _NativeResult(h, A.rows, A.cols, min(cfg.maxiter, A.cols) + 1)
    term = nr.info["termination"]
    if term == "trivial":
        return SolveResult(x=nr.x, trace=SolverTrace(), termination="trivial")
    trace = SolverTrace()
    for i in range(nr.info["n_records"]):
        rel = float(nr.relerr[i])
        trace.records.append(TraceRecord(
            iteration=i + 1, proj_obj=float(nr.proj[i]),
            rel_err=None if (x_true is None or np.isnan(rel)) else rel,
            res_norm=float(nr.resnorm[i]) if cfg.compute_diagnostics else None,
            kappa_basis=_opt(nr.kappa_basis[i]) if cfg.compute_diagnostics else None,
            matvecs=int(nr.matvecs[i]), tmatvecs=int(nr.tmatvecs[i]), dots=int(nr.dots[i]),
            sketches=0, wall_ms=float(nr.wall[i]), rank_fallback=bool(nr.rankfb[i]),
        ))
    return SolveResult(x=nr.x, trace=trace, termination=term, loop_ms=nr.loop_ms)


def gmres(A, b, cfg=None, x_true=None):
    """Arnoldi minimal-residual reference for square systems (solvers.py:256-325):
    Gram-Schmidt with one reorthogonalisation pass, tracked inner products,
    lucky breakdown at h_{k+1,k} <= 1e-14 |h|, lam^2 |y|^2 damping."""
    if not A.is_square:
        raise ValueError("gmres needs a square operator")
    return _krylov_solve(A, b, cfg, x_true, 0)


def lsqr(A, b, cfg=None, x_true=None):
    """Golub-Kahan least-squares reference (solvers.py:328-403), both sequences
    reorthogonalised; lam > 0 gives damped least squares on the Krylov space."""
    return _krylov_solve(A, b, cfg, x_true, 1)


def cmrh(A, b, cfg=None, x_true=None):
    """Quasi-minimal residual on the pivoted Hessenberg basis (solvers.py:542-550):
    min |beta e1 - H_{k+1,k} y| (+ lam^2 |y|^2), x = L_k y."""
    return _hessenberg_solve(A, b, cfg, x_true, True, False, sketched=False)


def lslu(A, b, cfg=None, x_true=None):
    """Quasi-minimal residual on the generalized Hessenberg bases (solvers.py:553-559)."""
    return _hessenberg_solve(A, b, cfg, x_true, False, False, sketched=False)


SOLVERS = {
    "gmres": gmres,
    "lsqr": lsqr,
    "cmrh": cmrh,
    "lslu": lslu,
    "scmrh": scmrh,
    "slslu": slslu,
}
