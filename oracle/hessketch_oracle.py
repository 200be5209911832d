"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference's sketched
Hessenberg (sCMRH) / sketched LSLU (sLSLU) iteration loop.

Every function cites the reference lines it restates (paths relative to the
reference package ``pkg/src/hessketch``).  The restatement is parametrised by
the working precision ``dtype``:

* ``np.float64`` -- the reference itself.  With the same operator callables and
  the same sketch matrices it reproduces the reference bit for bit (pinned by
  ``tests/test_oracle_golden.py`` against fixtures generated from the reference).
* ``storage="bfloat16"`` (with ``np.float32``) -- the basis columns are
  *stored* in bfloat16: each normalised column is rounded to nearest-even
  bf16 when it is appended, and everything that reads the basis afterwards
  (the operator input A l_k, the in-order elimination, x = L_k y) reads the
  stored values.  This is the device's bf16-storage path (BASELINE config 5:
  "basis vectors stored in bf16 with fp32 pivoting, axpy and sketch
  accumulation"); the reference has no counterpart.  Partial pivoting keeps
  the pivot entry exactly 1.0 and earlier pivot rows exactly 0.0 in bf16, so
  the coefficients read from u at the pivots are still the forward
  substitution on the stored pivot rows.
* ``np.float32`` -- "oracle32": identical algorithm, but the Krylov vectors
  (r0, u, q, basis columns) and the elimination / pivot / normalisation
  arithmetic are float32, as the device's fp32 path computes them.  Sketch
  products, the projected least-squares solve and the iterate x = L_k y stay in
  float64 (the device does the same).  The reference hard-casts to float64
  (linops.py:109,115,119,125; hessenberg.py:164,282; solvers.py:418), so this
  precision variant has no reference counterpart; it is pinned to the float64
  path on problems where both must agree (see tests).

Not a product path: nothing in ``paper_2502_02721_b200`` imports this module.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg
import scipy.sparse

RANK_TOL = 1e-14  # linops.py:36


class RankDeficiencyError(np.linalg.LinAlgError):
    """linops.py:39-50."""

    def __init__(self, message, rank):
        super().__init__(message)
        self.rank = rank


class TrivialSolution(Exception):
    """hessenberg.py:79-90."""

    def __init__(self, message, x):
        super().__init__(message)
        self.x = x


# ---------------------------------------------------------------------------
# operators (linops.py:53-149)


@dataclass
class Counters:
    """linops.py:53-68 (matvec, transpose, dot, sketch tallies)."""

    matvecs: int = 0
    tmatvecs: int = 0
    dots: int = 0
    sketches: int = 0

    def snapshot(self):
        return (self.matvecs, self.tmatvecs, self.dots, self.sketches)


class Operator:
    """Restates ``LinearOperator.apply``/``apply_transpose`` (linops.py:107-125):
    length check, one count per application, result cast to the working dtype."""

    def __init__(self, rows, cols, forward, transpose, dtype=np.float64):
        self.rows, self.cols = int(rows), int(cols)
        self.forward, self.transpose = forward, transpose
        self.dtype = np.dtype(dtype)
        self.counters = Counters()

    @property
    def is_square(self):
        return self.rows == self.cols

    def fresh(self):
        return Operator(self.rows, self.cols, self.forward, self.transpose, self.dtype)

    def apply(self, x):
        x = np.asarray(x, dtype=self.dtype)
        if x.shape != (self.cols,):
            raise ValueError(f"operator expects a vector of length {self.cols}")
        self.counters.matvecs += 1
        return np.asarray(self.forward(x), dtype=self.dtype)

    def apply_transpose(self, y):
        y = np.asarray(y, dtype=self.dtype)
        if y.shape != (self.rows,):
            raise ValueError(f"operator transpose expects a vector of length {self.rows}")
        self.counters.tmatvecs += 1
        return np.asarray(self.transpose(y), dtype=self.dtype)


def csr_operator(M, dtype=np.float64):
    """``LinearOperator.from_matrix`` on a sparse matrix (linops.py:137-141):
    forward ``M @ x`` and transpose ``M.T.tocsr() @ y``.  scipy's csr_matvec is
    a sequential left-to-right row sum without FMA; with float32 data and a
    float32 vector it runs in float32, with float64 it upcasts (exactly)."""
    M = scipy.sparse.csr_matrix(M)
    M.sort_indices()
    Mt = M.T.tocsr()
    if np.dtype(dtype) == np.float32:
        M = M.astype(np.float32)
        Mt = Mt.astype(np.float32)
    return Operator(M.shape[0], M.shape[1], lambda x: M @ x, lambda y: Mt @ y, dtype)


def dense_operator(M, dtype=np.float64, sequential=True):
    """``LinearOperator.from_matrix`` on a dense array (linops.py:142-145).

    The reference computes ``M @ x`` with BLAS dgemv, whose summation order is
    library-defined.  ``sequential=True`` pins the order to a left-to-right row
    sum without FMA (what the device dense kernel computes); ``False`` defers to
    numpy's BLAS, i.e. the reference itself."""
    M = np.asarray(M, dtype=dtype)
    if M.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    if not sequential:
        return Operator(M.shape[0], M.shape[1], lambda x: M @ x, lambda y: M.T @ y, dtype)
    Mt = np.ascontiguousarray(M.T)
    return Operator(
        M.shape[0], M.shape[1],
        lambda x: sequential_rows(M, x), lambda y: sequential_rows(Mt, y), dtype,
    )


def sequential_rows(M, x):
    """y_i = (((0 + M_i0 x_0) + M_i1 x_1) + ...) in M's dtype, no FMA."""
    M = np.asarray(M)
    x = np.asarray(x, dtype=M.dtype)
    acc = np.zeros(M.shape[0], dtype=M.dtype)
    for j in range(M.shape[1]):
        acc = acc + M[:, j] * x[j]
    return acc


def identity_operator(n, dtype=np.float64):
    """linops.py:147-149."""
    return Operator(n, n, lambda x: x.copy(), lambda y: y.copy(), dtype)


# ---------------------------------------------------------------------------
# pivoting (hessenberg.py:93-129)


def pivot_full(v, admissible):
    """Full-scan ``pivot_select`` (hessenberg.py:93-115): argmax |v| over the
    admissible set, ties to the smallest index, signed value; 0 => breakdown."""
    admissible = np.asarray(admissible, dtype=np.int64)
    if admissible.size == 0:
        raise ValueError("admissible index set is empty")
    mags = np.abs(v[admissible])
    top = mags.max()
    if top == 0.0:
        return int(admissible.min()), 0.0
    idx = int(admissible[mags == top].min())
    return idx, v[idx]


def pivot_select(v, admissible, sample_size=0, rng=None):
    """``pivot_select`` (hessenberg.py:93-115) with the sampled strategy:
    when ``0 < sample_size < len(admissible)`` the candidates are
    ``rng.choice(admissible, sample_size, replace=False)``."""
    admissible = np.asarray(admissible, dtype=np.int64)
    if admissible.size == 0:
        raise ValueError("admissible index set is empty")
    if sample_size and sample_size < admissible.size:
        admissible = rng.choice(admissible, size=sample_size, replace=False)
    return pivot_full(v, admissible)


def pivot_with_fallback(v, admissible, sample_size=0, rng=None):
    """hessenberg.py:118-124: a sampled miss (all zero) rescans everything."""
    idx, val = pivot_select(v, admissible, sample_size, rng)
    if val == 0.0 and sample_size:
        idx, val = pivot_full(v, admissible)
    return idx, val


def _swap_to_position(perm, used, idx):
    """hessenberg.py:127-129."""
    pos = used + int(np.nonzero(perm[used:] == idx)[0][0])
    perm[used], perm[pos] = perm[pos], perm[used]


# ---------------------------------------------------------------------------
# square process (hessenberg.py:132-226)


@dataclass
class SquareState:
    L: list
    h_cols: list
    t: np.ndarray
    beta: float
    k: int
    breakdown: bool
    r0: np.ndarray
    last_product: np.ndarray = None
    sample_size: int = 0
    rng: object = None

    def H_matrix(self, rows=None):
        k = len(self.h_cols)
        H = np.zeros((k + 1, k))
        for j, col in enumerate(self.h_cols):
            H[: j + 2, j] = col
        return H if rows is None else H[:rows]


def round_bf16(a):
    """Round float32 values to the nearest bfloat16 (ties to even), returned as
    float32 -- the device's __float2bfloat16_rn storage conversion."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    bits = a.view(np.uint32).astype(np.uint64)
    bits = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    return bits.astype(np.uint32).view(np.float32)


def _store(v, storage):
    """A new basis column as the basis stores it."""
    return round_bf16(v) if storage == "bfloat16" else v


def init_square(A, b, x0=None, sample_size=0, rng=None, storage=None):
    """hessenberg.py:160-188 (full or sampled pivoting)."""
    if not A.is_square:
        raise ValueError("the square Hessenberg process needs a square operator")
    dt = A.dtype
    b = np.asarray(b, dtype=dt)
    if b.shape != (A.rows,):
        raise ValueError(f"b must have length {A.rows}")
    r0 = b.copy() if x0 is None else b - A.apply(np.asarray(x0, dtype=dt))
    t = np.arange(A.rows)
    idx, beta = pivot_with_fallback(r0, t, sample_size, rng)
    if beta == 0.0:
        x = np.zeros(A.cols) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
        raise TrivialSolution("initial residual is zero; starting point is exact", x)
    _swap_to_position(t, 0, idx)
    st = SquareState([_store(r0 / beta, storage)], [], t, beta, 0, False, r0)
    st.sample_size, st.rng = sample_size, rng
    st.storage = storage
    return st


def _eliminate(u, basis, perm, k):
    """The in-order elimination of hessenberg.py:209-212 / 347-350 / 371-374:
    c_j = u[perm_j]; u <- u - c_j * basis_j (product rounded, then difference)."""
    h = np.empty(k + 1)
    for j in range(k):
        c = u[perm[j]]
        h[j] = c
        u = u - c * basis[j]
    return u, h


def step_square(state, A, keep_product=True):
    """hessenberg.py:191-226."""
    if state.breakdown:
        raise RuntimeError("factorization already broke down")
    k = state.k + 1
    n = A.rows
    u = A.apply(state.L[-1])
    if keep_product:
        state.last_product = u.copy()
    u, h = _eliminate(u, state.L, state.t, k)
    if k < n:
        idx, val = pivot_with_fallback(u, state.t[k:], state.sample_size, state.rng)
    else:
        val = 0.0
    if val == 0.0:
        h[k] = 0.0
        state.breakdown = True
    else:
        h[k] = val
        _swap_to_position(state.t, k, idx)
        state.L.append(_store(u / val, getattr(state, "storage", None)))
    state.h_cols.append(h)
    state.k = k
    return state


# ---------------------------------------------------------------------------
# generalized process (hessenberg.py:229-390)


@dataclass
class GenState:
    D: list
    L: list
    h_cols: list
    w_cols: list
    t: np.ndarray
    g: np.ndarray
    beta: float
    alpha: float
    k: int
    breakdown: bool
    r0: np.ndarray
    last_data_product: np.ndarray = None
    last_solution_product: np.ndarray = None
    sample_size: int = 0
    rng: object = None

    def H_matrix(self, rows=None):
        k = len(self.h_cols)
        H = np.zeros((k + 1, k))
        for j, col in enumerate(self.h_cols):
            H[: j + 2, j] = col
        return H if rows is None else H[:rows]

    def W_matrix(self, rows=None):
        cols = len(self.w_cols)
        W = np.zeros((cols, cols))
        for j, col in enumerate(self.w_cols):
            W[: j + 1, j] = col
        return W if rows is None else W[:rows]


def init_generalized(A, b, x0=None, sample_size=0, rng=None, storage=None):
    """hessenberg.py:275-326 (full or sampled pivoting)."""
    dt = A.dtype
    b = np.asarray(b, dtype=dt)
    if b.shape != (A.rows,):
        raise ValueError(f"b must have length {A.rows}")
    r0 = b.copy() if x0 is None else b - A.apply(np.asarray(x0, dtype=dt))
    zero_x = np.zeros(A.cols) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    t = np.arange(A.rows)
    idx, beta = pivot_with_fallback(r0, t, sample_size, rng)
    if beta == 0.0:
        raise TrivialSolution("initial residual is zero; starting point is exact", zero_x)
    d1 = _store(r0 / beta, storage)
    _swap_to_position(t, 0, idx)
    v0 = A.apply_transpose(r0)
    g = np.arange(A.cols)
    idx2, alpha = pivot_with_fallback(v0, g, sample_size, rng)
    if alpha == 0.0:
        raise TrivialSolution(
            "transposed residual is zero; the normal equations already hold", zero_x
        )
    l1 = _store(v0 / alpha, storage)
    _swap_to_position(g, 0, idx2)
    r = A.apply_transpose(d1)
    st = GenState([d1], [l1], [], [np.array([r[g[0]]], dtype=np.float64)], t, g,
                  beta, alpha, 0, False, r0)
    st.last_solution_product = r.copy()
    st.sample_size, st.rng = sample_size, rng
    st.storage = storage
    return st


def step_generalized(state, A, keep_products=True):
    """hessenberg.py:329-390."""
    if state.breakdown:
        raise RuntimeError("factorization already broke down")
    k = state.k + 1
    m, n = A.rows, A.cols
    u = A.apply(state.L[-1])
    if keep_products:
        state.last_data_product = u.copy()
    u, h = _eliminate(u, state.D, state.t, k)
    if k < m:
        idx, val = pivot_with_fallback(u, state.t[k:], state.sample_size, state.rng)
    else:
        val = 0.0
    if val == 0.0:
        h[k] = 0.0
        state.h_cols.append(h)
        state.k = k
        state.breakdown = True
        return state
    h[k] = val
    _swap_to_position(state.t, k, idx)
    d_new = _store(u / val, getattr(state, "storage", None))
    state.D.append(d_new)
    state.h_cols.append(h)

    q = A.apply_transpose(d_new)
    if keep_products:
        state.last_solution_product = q.copy()
    q, w = _eliminate(q, state.L, state.g, k)
    if k < n:
        idx2, val2 = pivot_with_fallback(q, state.g[k:], state.sample_size, state.rng)
    else:
        val2 = 0.0
    if val2 == 0.0:
        w[k] = 0.0
        state.w_cols.append(w)
        state.k = k
        state.breakdown = True
        return state
    w[k] = val2
    _swap_to_position(state.g, k, idx2)
    state.L.append(_store(q / val2, getattr(state, "storage", None)))
    state.w_cols.append(w)
    state.k = k
    return state


# ---------------------------------------------------------------------------
# sketches (sketch.py:43-65, 115-123)


def gaussian_sketch_entries(out_rows, in_rows, seed):
    """``make_gaussian_sketch`` (sketch.py:43-53): PCG64(seed) standard normals,
    row-major (out_rows, in_rows), divided by sqrt(out_rows)."""
    if out_rows < 1 or in_rows < 1:
        raise ValueError("sketch dimensions must be positive")
    gen = np.random.Generator(np.random.PCG64(seed))
    return gen.standard_normal((out_rows, in_rows)) / np.sqrt(out_rows)


def derive_seed(seed, stream):
    """sketch.py:115-123."""
    ss = np.random.SeedSequence(int(seed), spawn_key=(int(stream),))
    return int(ss.generate_state(1, dtype=np.uint64)[0])


def sketch_apply(S, v, counters):
    """sketch.py:56-65: ``S @ v`` (float64) plus one sketch count."""
    counters.sketches += 1
    return np.asarray(S @ np.asarray(v, dtype=np.float64), dtype=np.float64)


# ---------------------------------------------------------------------------
# projected least squares (linops.py:168-229, solvers.py:204-225)


def dense_qr_ls(M, rhs):
    """linops.py:168-207: column-pivoted economic QR, rank gate, trsv."""
    M = np.asarray(M, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    l, k = M.shape
    if l < k:
        raise ValueError("need at least as many rows as columns")
    Q, R, piv = scipy.linalg.qr(M, mode="economic", pivoting=True)
    diag = np.abs(np.diag(R))
    largest = diag.max() if k else 0.0
    if largest == 0.0 or diag.min() < RANK_TOL * largest:
        rank = int(np.count_nonzero(diag >= RANK_TOL * largest)) if largest else 0
        raise RankDeficiencyError("rank deficient", rank)
    y_perm = scipy.linalg.solve_triangular(R, Q.T @ rhs)
    y = np.empty(k)
    y[piv] = y_perm
    return y


def stacked_tikhonov_ls(M, N, rhs, lam):
    """linops.py:210-229: QR of [M; lam N] against [rhs; 0]; lam = 0 is dense_qr_ls."""
    if lam == 0.0:
        return dense_qr_ls(M, rhs)
    stacked = np.vstack([M, lam * N])
    srhs = np.concatenate([rhs, np.zeros(N.shape[0])])
    return dense_qr_ls(stacked, srhs)


def projected_solve(M, rhs, lam, N=None):
    """solvers.py:204-218 (truncated lstsq fallback on rank deficiency)."""
    try:
        if lam == 0.0:
            return dense_qr_ls(M, rhs), False
        return stacked_tikhonov_ls(M, N, rhs, lam), False
    except RankDeficiencyError:
        if lam == 0.0:
            stacked, srhs = M, rhs
        else:
            stacked = np.vstack([M, lam * N])
            srhs = np.concatenate([rhs, np.zeros(N.shape[0])])
        y, _, _, _ = np.linalg.lstsq(stacked, srhs, rcond=None)
        return y, True


def objective(M, rhs, y, lam, N=None):
    """solvers.py:221-225."""
    val = np.linalg.norm(M @ y - rhs) ** 2
    if lam > 0.0:
        val += lam**2 * np.linalg.norm(N @ y) ** 2
    return float(np.sqrt(val))


# ---------------------------------------------------------------------------
# the loop driver (solvers.py:410-539, sketched branch)


@dataclass
class Result:
    x: np.ndarray
    records: list
    termination: str
    state: object = None
    Z: np.ndarray = None
    F: np.ndarray = None
    sr0: np.ndarray = None
    loop_seconds: float = 0.0

    def column(self, name):
        return [r[name] for r in self.records]


def hessenberg_solve(
    A, b, *, square, maxiter, ell=None, lam=0.0, seed=0, S2=None, S1=None,
    x0=None, x_true=None, sketch_basis=False, sketched=True, pivot_sample=0, pivot_seed=0, printed_f=False,
    storage=None,
):
    """Restates ``_hessenberg_solve`` (solvers.py:410-539) for the sketched
    solvers ``scmrh`` / ``slslu`` / ``*_tikhonov`` (solvers.py:562-605) and,
    with ``sketched=False``, the unsketched ``cmrh`` / ``lslu``
    (solvers.py:542-559: projected problem H_{k+1,k} y ~ beta e1, plus
    lam^2 |y|^2).  ``pivot_sample`` > 0 selects sampled pivoting
    (``PivotStrategy.sampled(pivot_sample, pivot_seed)``, hessenberg.py:48-73).

    ``S2`` / ``S1``: explicit sketch matrices (anything supporting ``@``).  When
    None they are drawn exactly as the reference draws them
    (``make_gaussian_sketch(ell, A.rows, seed)`` and
    ``make_gaussian_sketch(ell, A.cols, derive_seed(seed, 1))``, solvers.py:452-459).
    Returns a :class:`Result` with per-iteration records carrying the
    reference's TraceRecord fields.
    """
    if square and not A.is_square:
        raise ValueError("this solver needs a square operator")
    A = A.fresh()
    c = A.counters
    init = init_square if square else init_generalized
    rng = np.random.default_rng(pivot_seed) if pivot_sample else None
    try:
        state = init(A, b, x0=x0, sample_size=pivot_sample, rng=rng, storage=storage)
    except TrivialSolution as sig:
        return Result(x=sig.x, records=[], termination="trivial")
    if not sketched:
        return _unsketched_loop(A, c, state, square, maxiter, lam, x0, x_true)

    if S2 is not None:
        if S2.shape[1] != A.rows:
            raise ValueError("sketch/operator length mismatch")
        ell = S2.shape[0]
    elif ell is None:
        ell = 10 * (maxiter + 1)  # solvers.py:113-116
    if ell < maxiter + 1:  # solvers.py:447-451
        raise ValueError(f"sketch_rows={ell} cannot embed a {maxiter}-dimensional projected problem")
    if S2 is None:
        S2 = gaussian_sketch_entries(ell, A.rows, seed)
    keep = not sketch_basis
    sr0 = sketch_apply(S2, state.r0, c)
    Z_cols, G_cols, F_cols = [], [], []
    if sketch_basis:
        first = state.L[0] if square else state.D[0]
        G_cols.append(sketch_apply(S2, first, c))
    if lam > 0.0:
        if S1 is None:
            S1 = gaussian_sketch_entries(ell, A.cols, derive_seed(seed, 1))
        # printed_f: slslu_tikhonov(printed_f_columns=True) sketches the
        # unreduced transpose products (solvers.py:460-461, 488-490)
        f0 = state.last_solution_product if (printed_f and not square) else state.L[0]
        F_cols.append(sketch_apply(S1, f0, c))

    records = []
    termination = "maxiter"
    x = None
    x0_64 = None if x0 is None else np.asarray(x0, dtype=np.float64)
    tic_all = time.perf_counter()
    for k in range(1, maxiter + 1):
        tic = time.perf_counter()
        n_basis_before = len(state.L) if square else len(state.D)
        n_sol_before = len(state.L)
        if square:
            step_square(state, A, keep_product=keep)
            prod = state.last_product
        else:
            step_generalized(state, A, keep_products=keep)
            prod = state.last_data_product
        if keep:
            Z_cols.append(sketch_apply(S2, prod, c))
        else:
            cols = state.L if square else state.D
            if len(cols) > n_basis_before:
                G_cols.append(sketch_apply(S2, cols[-1], c))
        if lam > 0.0:
            if printed_f and not square:
                if len(state.D) > n_basis_before:
                    F_cols.append(sketch_apply(S1, state.last_solution_product, c))
            elif len(state.L) > n_sol_before:
                F_cols.append(sketch_apply(S1, state.L[-1], c))

        Lk = np.column_stack(state.L[:k]).astype(np.float64)
        if sketch_basis:
            G = np.column_stack(G_cols)
            M = G @ state.H_matrix(rows=G.shape[1])
        else:
            M = np.column_stack(Z_cols)
        N = np.column_stack(F_cols[:k]) if lam > 0.0 else None
        y, fallback = projected_solve(M, sr0, lam, N)
        x = Lk @ y
        if x0_64 is not None:
            x = x0_64 + x
        rec = dict(
            iteration=k,
            proj_obj=objective(M, sr0, y, lam, N),
            sres_norm=float(np.linalg.norm(M @ y - sr0)),
            rel_err=None,
            rank_fallback=fallback,
        )
        if x_true is not None:
            xt = np.asarray(x_true, dtype=np.float64)
            rec["rel_err"] = float(np.linalg.norm(x - xt) / np.linalg.norm(xt))
        rec["matvecs"], rec["tmatvecs"], rec["dots"], rec["sketches"] = c.snapshot()
        rec["wall_ms"] = (time.perf_counter() - tic) * 1e3
        records.append(rec)
        if state.breakdown:
            termination = "breakdown"
            break
    loop_s = time.perf_counter() - tic_all
    return Result(
        x=x, records=records, termination=termination, state=state,
        Z=np.column_stack(Z_cols) if Z_cols else None,
        F=np.column_stack(F_cols) if F_cols else None, sr0=sr0, loop_seconds=loop_s,
    )


def _unsketched_loop(A, c, state, square, maxiter, lam, x0, x_true):
    """solvers.py:468-539 with ``sketched=False``: M = H_{k+1,k}, rhs = beta e1,
    N = I_k when lam > 0; no sketch is applied and sres_norm stays None."""
    records = []
    termination = "maxiter"
    x = None
    x0_64 = None if x0 is None else np.asarray(x0, dtype=np.float64)
    tic_all = time.perf_counter()
    for k in range(1, maxiter + 1):
        tic = time.perf_counter()
        if square:
            step_square(state, A, keep_product=False)
        else:
            step_generalized(state, A, keep_products=False)
        Lk = np.column_stack(state.L[:k]).astype(np.float64)
        M = state.H_matrix()
        rhs = np.zeros(M.shape[0])
        rhs[0] = state.beta
        N = np.eye(k) if lam > 0.0 else None
        y, fallback = projected_solve(M, rhs, lam, N)
        x = Lk @ y
        if x0_64 is not None:
            x = x0_64 + x
        rec = dict(iteration=k, proj_obj=objective(M, rhs, y, lam, N), sres_norm=None, rel_err=None,
                   rank_fallback=fallback)
        if x_true is not None:
            xt = np.asarray(x_true, dtype=np.float64)
            rec["rel_err"] = float(np.linalg.norm(x - xt) / np.linalg.norm(xt))
        rec["matvecs"], rec["tmatvecs"], rec["dots"], rec["sketches"] = c.snapshot()
        rec["wall_ms"] = (time.perf_counter() - tic) * 1e3
        records.append(rec)
        if state.breakdown:
            termination = "breakdown"
            break
    return Result(x=x, records=records, termination=termination, state=state,
                  loop_seconds=time.perf_counter() - tic_all)


def pivots_of(state):
    """Pivot sequences actually used: t[:len(basis)], g[:len(L)]."""
    if isinstance(state, GenState):
        return state.t[: len(state.D)].copy(), state.g[: len(state.L)].copy()
    return state.t[: len(state.L)].copy(), None


# ---------------------------------------------------------------------------
# the reference's comparison solvers (solvers.py:256-403), restated


def _tracked_dot(c, x, y):
    """linops.py:152-159: one charge per inner product."""
    c.dots += 1
    return float(np.dot(x, y))


def _tracked_norm(c, x):
    """linops.py:162-165: a norm costs one inner product."""
    c.dots += 1
    return float(np.linalg.norm(x))


def _krylov_record(k, M, rhs, y, lam, N, fallback, x, x_true, A, b, diagnostics, c, tic):
    rec = dict(iteration=k, proj_obj=objective(M, rhs, y, lam, N), sres_norm=None, rel_err=None,
               rank_fallback=fallback, res_norm=None)
    if x_true is not None:
        xt = np.asarray(x_true, dtype=np.float64)
        rec["rel_err"] = float(np.linalg.norm(x - xt) / np.linalg.norm(xt))
    if diagnostics:  # raw forward application, not counted (solvers.py:247-250)
        rec["res_norm"] = float(np.linalg.norm(np.asarray(b, dtype=float) - np.asarray(A.forward(x), dtype=float)))
    rec["wall_ms"] = (time.perf_counter() - tic) * 1e3
    return rec


def gmres(A, b, *, maxiter, lam=0.0, x0=None, x_true=None, diagnostics=False):
    """solvers.py:256-325: Arnoldi, modified Gram-Schmidt + one
    reorthogonalisation pass, lucky breakdown h_{k+1,k} <= 1e-14 |h|."""
    if not A.is_square:
        raise ValueError("gmres needs a square operator")
    A = A.fresh()
    c = A.counters
    b = np.asarray(b, dtype=float)
    x0 = None if x0 is None else np.asarray(x0, dtype=float)
    r0 = b.copy() if x0 is None else b - A.apply(x0)
    beta = _tracked_norm(c, r0)
    if beta == 0.0:
        return Result(x=np.zeros(A.cols) if x0 is None else x0.copy(), records=[], termination="trivial")
    V = [r0 / beta]
    h_cols = []
    records = []
    x = None
    termination = "maxiter"
    for k in range(1, min(maxiter, A.rows) + 1):
        tic = time.perf_counter()
        w = A.apply(V[-1])
        h = np.empty(k + 1)
        for j in range(k):
            h[j] = _tracked_dot(c, V[j], w)
            w = w - h[j] * V[j]
        for j in range(k):
            corr = _tracked_dot(c, V[j], w)
            w = w - corr * V[j]
            h[j] += corr
        h[k] = _tracked_norm(c, w)
        h_cols.append(h)
        lucky = h[k] <= 1e-14 * np.linalg.norm(h)
        if not lucky:
            V.append(w / h[k])
        H = np.zeros((k + 1, k))
        for j, col in enumerate(h_cols):
            H[: j + 2, j] = col
        rhs = np.zeros(k + 1)
        rhs[0] = beta
        N = np.eye(k) if lam > 0.0 else None
        y, fallback = projected_solve(H, rhs, lam, N)
        x = np.column_stack(V[:k]) @ y
        if x0 is not None:
            x = x0 + x
        rec = _krylov_record(k, H, rhs, y, lam, N, fallback, x, x_true, A, b, diagnostics, c, tic)
        rec["matvecs"], rec["tmatvecs"], rec["dots"], rec["sketches"] = c.snapshot()
        records.append(rec)
        if lucky:
            termination = "breakdown"
            break
    return Result(x=x, records=records, termination=termination)


def lsqr(A, b, *, maxiter, lam=0.0, x0=None, x_true=None, diagnostics=False):
    """solvers.py:328-403: Golub-Kahan with one reorthogonalisation pass on
    both sequences; exhausted when beta <= 1e-14 alpha or alpha <= 1e-14 beta."""
    A = A.fresh()
    c = A.counters
    b = np.asarray(b, dtype=float)
    x0 = None if x0 is None else np.asarray(x0, dtype=float)
    r0 = b.copy() if x0 is None else b - A.apply(x0)
    zero = np.zeros(A.cols) if x0 is None else x0.copy()
    beta1 = _tracked_norm(c, r0)
    if beta1 == 0.0:
        return Result(x=zero, records=[], termination="trivial")
    U = [r0 / beta1]
    z = A.apply_transpose(U[0])
    alpha = _tracked_norm(c, z)
    if alpha == 0.0:
        return Result(x=zero, records=[], termination="trivial")
    V = [z / alpha]
    alphas, betas = [alpha], []
    records = []
    x = None
    termination = "maxiter"
    for k in range(1, min(maxiter, A.cols) + 1):
        tic = time.perf_counter()
        w = A.apply(V[-1]) - alphas[-1] * U[-1]
        for u in U:
            w = w - _tracked_dot(c, u, w) * u
        beta = _tracked_norm(c, w)
        exhausted = beta <= 1e-14 * alphas[-1]
        if not exhausted:
            U.append(w / beta)
        betas.append(beta)
        B = np.zeros((k + 1, k))
        for j in range(k):
            B[j, j] = alphas[j]
            B[j + 1, j] = betas[j]
        rhs = np.zeros(k + 1)
        rhs[0] = beta1
        N = np.eye(k) if lam > 0.0 else None
        y, fallback = projected_solve(B, rhs, lam, N)
        x = np.column_stack(V[:k]) @ y
        if x0 is not None:
            x = x0 + x
        rec = _krylov_record(k, B, rhs, y, lam, N, fallback, x, x_true, A, b, diagnostics, c, tic)
        if not exhausted:
            z = A.apply_transpose(U[-1]) - beta * V[-1]
            for v in V:
                z = z - _tracked_dot(c, v, z) * v
            alpha = _tracked_norm(c, z)
            if alpha <= 1e-14 * beta:
                exhausted = True
            else:
                V.append(z / alpha)
                alphas.append(alpha)
        rec["matvecs"], rec["tmatvecs"], rec["dots"], rec["sketches"] = c.snapshot()
        records.append(rec)
        if exhausted:
            termination = "breakdown"
            break
    return Result(x=x, records=records, termination=termination)
