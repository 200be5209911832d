"""Pivoting strategy and factorization state of the pivoted Hessenberg
processes (hessenberg.py:48-390 of the reference), as seen from the host.

The processes run on the device: inside ``hs_solve`` (what comes back is a
:class:`DeviceFactorization` exposing the reference state's fields ``t``,
``g``, ``k``, ``breakdown``, ``L_cols``, ``D_cols``, ``H_matrix()``,
``W_matrix()``, ``L_matrix()``, ``D_matrix()``), or one step per call through
the reference's step-level API -- ``init_square`` / ``step_square``
(hessenberg.py:160-226) and ``init_generalized`` / ``step_generalized``
(hessenberg.py:275-390) -- whose state objects keep the factorization on the
device between calls (``hs_stepper_*``).  Basis columns are copied from the
device only when accessed.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

__all__ = [
    "PivotStrategy",
    "TrivialSolution",
    "DeviceFactorization",
    "HessenbergState",
    "GeneralizedHessenbergState",
    "init_square",
    "step_square",
    "init_generalized",
    "step_generalized",
    "dump_factorization",
    "pivot_select",
]


@dataclass(frozen=True)
class PivotStrategy:
    """hessenberg.py:48-73.  Only ``full`` runs on the device in this version."""

    kind: str = "full"
    sample_size: int = 0
    seed: int = 0

    def __post_init__(self):
        if self.kind not in ("full", "sampled"):
            raise ValueError(f"unknown pivot kind {self.kind!r}")
        if self.kind == "sampled" and self.sample_size < 1:
            raise ValueError("sampled pivoting needs sample_size >= 1")

    @classmethod
    def full(cls):
        return cls("full")

    @classmethod
    def sampled(cls, sample_size, seed=0):
        return cls("sampled", sample_size, seed)


class TrivialSolution(Exception):
    """hessenberg.py:79-90."""

    def __init__(self, message, x):
        super().__init__(message)
        self.x = x


def _full_permutation(size, pivots):
    """Replay hessenberg.py:127-129 swaps: position k takes pivot k."""
    perm = np.arange(size)
    where = np.arange(size)  # where[v] = position of value v
    for k, idx in enumerate(pivots):
        pos = where[idx]
        other = perm[k]
        perm[k], perm[pos] = idx, other
        where[idx], where[other] = k, pos
    return perm


class _LazyCols:
    def __init__(self, fetch, count):
        self._fetch = fetch
        self._count = count
        self._cache = {}

    def __len__(self):
        return self._count

    def __getitem__(self, j):
        if isinstance(j, slice):
            return [self[i] for i in range(*j.indices(self._count))]
        if j < 0:
            j += self._count
        if not 0 <= j < self._count:
            raise IndexError(j)
        if j not in self._cache:
            self._cache[j] = self._fetch(j)
        return self._cache[j]

    def __iter__(self):
        for j in range(self._count):
            yield self[j]


class DeviceFactorization:
    """Host view of the device factorization A L_k = L_{k+1} H (square) or
    A L_k = D_{k+1} H, A^T D_{k+1} = L_{k+1} W (rectangular)."""

    def __init__(self, result, square, rows, cols, basis_rows=None):
        from . import _lib

        self._res = result  # keeps the native result (and device bases) alive
        self.square = square
        info = result.info
        self.k = info["k"]
        self.breakdown = info["termination"] == "breakdown"
        self._t = result.pivots_t
        self._g = result.pivots_g
        self._rows, self._cols = rows, cols
        self._H = result.H
        self._W = result.W

        def fetch(which, length):
            def f(j):
                out = np.empty(length)
                _lib.check(_lib.load().hs_result_basis(result.handle, which, int(j), _lib.ptr(out)))
                return out
            return f

        # basis_rows: (data, solution) rows held here -- this rank's shard of a
        # row-sharded solve (hs_dist.inc), the full length otherwise
        d_len, l_len = basis_rows if basis_rows is not None else (rows, cols)
        self.L_cols = _LazyCols(fetch(0, l_len), info["n_basis_sol"])
        self.D_cols = None if square else _LazyCols(fetch(1, d_len), info["n_basis_data"])
        self._tfull = None
        self._gfull = None

    @property
    def t(self):
        if self._tfull is None:
            self._tfull = _full_permutation(self._rows, self._t)
        return self._tfull

    @property
    def g(self):
        if self.square:
            raise AttributeError("square factorizations have no g")
        if self._gfull is None:
            self._gfull = _full_permutation(self._cols, self._g)
        return self._gfull

    def H_matrix(self, rows=None):
        return self._H if rows is None else self._H[:rows]

    def W_matrix(self, rows=None):
        if self.square:
            raise AttributeError("square factorizations have no W")
        return self._W if rows is None else self._W[:rows]

    def L_matrix(self):
        return np.column_stack(list(self.L_cols))

    def D_matrix(self):
        if self.square:
            raise AttributeError("square factorizations have no D")
        return np.column_stack(list(self.D_cols))


def pivot_select(v, admissible, strategy, rng=None):
    """hessenberg.py:93-115 on the device: ``(index, signed value)`` of the
    largest |v| over the admissible rows, ties toward the smallest row index;
    value 0.0 means every candidate was zero.  With a sampled strategy the
    candidates are ``rng.choice(admissible, sample_size, replace=False)``
    drawn here, as the reference draws them."""
    from . import _lib

    admissible = np.asarray(admissible, dtype=int)
    if admissible.size == 0:
        raise ValueError("admissible index set is empty")
    if strategy.kind == "sampled" and strategy.sample_size < admissible.size:
        if rng is None:
            raise ValueError("sampled pivoting requires a random generator")
        admissible = rng.choice(admissible, size=strategy.sample_size, replace=False)
    v = np.ascontiguousarray(v, dtype=np.float64)
    cand = np.ascontiguousarray(admissible, dtype=np.int64)
    idx, val = _lib.c_i64(), _lib.c_dbl()
    _lib.check(_lib.load().hs_pivot_select(_lib.context().handle, v.size, _lib.ptr(v), cand.size, _lib.ptr(cand),
                                           ctypes.byref(idx), ctypes.byref(val)))
    return int(idx.value), float(val.value)


# ---------------------------------------------------------------------------
# step-level API (hessenberg.py:130-390)

_DTYPES = {"float64": (0, 0), "float32": (1, 1), "bfloat16": (1, 2)}


class _StepperState:
    """Device-resident state shared by the square and rectangular processes."""

    def __init__(self, handle, A, square, strategy, rng):
        self._h = handle
        self._square = square
        self.strategy = strategy
        self.rng = rng
        self._rows, self._cols = A.rows, A.cols
        self._op = A
        self.h_cols = []
        self.w_cols = []
        self.last_product = None
        self.last_data_product = None
        self.last_solution_product = None
        self._refresh()
        from . import _lib

        r0 = np.empty(A.rows)
        _lib.check(_lib.load().hs_stepper_r0(self._h, _lib.ptr(r0)))
        self.r0 = r0

    def _refresh(self):
        from . import _lib

        k, bd, side, nl, nd = (_lib.c_i32() for _ in range(5))
        beta, alpha = _lib.c_dbl(), _lib.c_dbl()
        _lib.check(_lib.load().hs_stepper_info(self._h, *(ctypes.byref(v) for v in (k, bd, side, nl, nd, beta, alpha))))
        self.k, self.breakdown = k.value, bool(bd.value)
        self._n_L, self._n_D = nl.value, nd.value
        self.beta, self.alpha = beta.value, alpha.value
        lib = _lib.load()
        tbuf = np.empty(max(self._n_D, 1), dtype=np.int64)
        gbuf = np.empty(max(self._n_L, 1), dtype=np.int64)
        _lib.check(lib.hs_stepper_pivots(self._h, _lib.ptr(tbuf), None if self._square else _lib.ptr(gbuf)))
        self._tp = tbuf[: self._n_D].copy()
        self._gp = None if self._square else gbuf[: self._n_L].copy()
        self._H = np.empty((self.k + 1, self.k)) if self.k else np.zeros((1, 0))
        Wc = None if self._square else np.empty((self._n_D, self._n_D))
        Hc = np.empty((self.k, self.k + 1)) if self.k else None
        _lib.check(lib.hs_stepper_hessenberg(self._h, None if Hc is None else _lib.ptr(Hc),
                                             None if Wc is None else _lib.ptr(Wc)))
        if Hc is not None:
            self._H = np.ascontiguousarray(Hc.T)
        if Wc is not None:
            self._W = np.ascontiguousarray(Wc.T)
        # per-column views in the reference's list form
        self.h_cols = [self._H[: j + 2, j].copy() for j in range(self.k)]
        if not self._square:
            self.w_cols = [self._W[: j + 1, j].copy() for j in range(self._n_D)]

        def fetch(which, length):
            def f(j):
                out = np.empty(length)
                _lib.check(_lib.load().hs_stepper_basis(self._h, which, int(j), _lib.ptr(out)))
                return out
            return f

        self.L_cols = _LazyCols(fetch(0, self._cols), self._n_L)
        if not self._square:
            self.D_cols = _LazyCols(fetch(1, self._rows), self._n_D)

    @property
    def t(self):
        """Swap-ordered pivot permutation (t[:k] = the pivots, hessenberg.py:127-129)."""
        return _full_permutation(self._rows, self._tp)

    def H_matrix(self, rows=None):
        return self._H if rows is None else self._H[:rows]

    def L_matrix(self):
        return np.column_stack(list(self.L_cols))

    def _positions(self, slots):
        """The reference's draws for this call: rng.choice(len(admissible), s)
        for each selection slot whose population exceeds s (hessenberg.py:106-109)."""
        if self.strategy.kind != "sampled":
            return None
        s = int(self.strategy.sample_size)
        out = np.full((len(slots), s), -1, dtype=np.int64)
        for i, pop in enumerate(slots):
            if pop > 0 and s < pop:
                out[i] = self.rng.choice(pop, size=s, replace=False)
        return out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None:
            try:
                from . import _lib

                _lib.load().hs_stepper_destroy(h)
            except Exception:
                pass
            self._h = None


class HessenbergState(_StepperState):
    """hessenberg.py:132-158: A L_k = L_{k+1} H_{k+1,k}, resident on the device."""


class GeneralizedHessenbergState(_StepperState):
    """hessenberg.py:229-272: A L_k = D_{k+1} H, A^T D_{k+1} = L_{k+1} W."""

    @property
    def g(self):
        return _full_permutation(self._cols, self._gp)

    def D_matrix(self):
        return np.column_stack(list(self.D_cols))

    def W_matrix(self, rows=None):
        return self._W if rows is None else self._W[:rows]


def _create(A, b, x0, strategy, square, dtype, capacity):
    from . import _lib
    from .linops import to_device_operator

    if dtype not in _DTYPES:
        raise ValueError(f"dtype must be one of {sorted(_DTYPES)}")
    dev = to_device_operator(A)
    b = np.asarray(b, dtype=float)
    if b.shape != (A.rows,):
        raise ValueError(f"b must have length {A.rows}, got shape {b.shape}")
    b = np.ascontiguousarray(b)
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=float)
    rng = np.random.default_rng(strategy.seed) if strategy.kind == "sampled" else None
    s = int(strategy.sample_size) if strategy.kind == "sampled" else 0
    pos = None
    if s:
        pops = [A.rows] if square else [A.rows, A.cols]
        pos = np.full((len(pops), s), -1, dtype=np.int64)
        for i, pop in enumerate(pops):
            if pop > 0 and s < pop:
                pos[i] = rng.choice(pop, size=s, replace=False)
    work, basis = _DTYPES[dtype]
    trivial = _lib.c_i32()
    h = _lib.c_vp()
    _lib.check(_lib.load().hs_stepper_create(dev.ctx.handle, dev.handle, 1 if square else 0, work, basis,
                                             int(capacity), _lib.ptr(b), _lib.ptr(x0a), s, _lib.ptr(pos),
                                             ctypes.byref(trivial), ctypes.byref(h)))
    counters = getattr(A, "counters", None)
    if counters is not None:
        if x0 is not None:
            counters.matvec_count += 1
        if not square and trivial.value != 1:
            counters.transpose_matvec_count += 1 if trivial.value == 2 else 2
    if trivial.value:
        x = np.zeros(A.cols) if x0 is None else np.asarray(x0, dtype=float).copy()
        msg = ("initial residual is zero; starting point is exact" if trivial.value == 1
               else "transposed residual is zero; the normal equations already hold")
        raise TrivialSolution(msg, x)
    cls = HessenbergState if square else GeneralizedHessenbergState
    return cls(h, A, square, strategy, rng)


def init_square(A, b, x0=None, strategy=PivotStrategy.full(), *, dtype="float64", capacity=64):
    """hessenberg.py:160-188 on the device.  ``dtype``: "float64" (the
    reference's arithmetic), "float32" or "bfloat16" (fp32 work, bf16 basis)."""
    if not A.is_square:
        raise ValueError("the square Hessenberg process needs a square operator")
    return _create(A, b, x0, strategy, True, dtype, capacity)


def init_generalized(A, b, x0=None, strategy=PivotStrategy.full(), *, dtype="float64", capacity=64):
    """hessenberg.py:275-326 on the device."""
    return _create(A, b, x0, strategy, False, dtype, capacity)


def _step(state, A, keep, square):
    from . import _lib

    if state.breakdown:
        raise RuntimeError("factorization already broke down")
    k = state.k + 1
    slots = [A.rows - k] if square else [A.rows - k, A.cols - k]
    pos = state._positions(slots)
    _lib.check(_lib.load().hs_stepper_step(state._h, 1 if keep else 0, _lib.ptr(pos)))
    nd_before = state._n_D
    state._refresh()
    counters = getattr(A, "counters", None)
    if counters is not None:
        counters.matvec_count += 1
        if not square and state._n_D > nd_before:
            counters.transpose_matvec_count += 1
    if keep:
        if square:
            state.last_product = np.empty(A.rows)
            _lib.check(_lib.load().hs_stepper_product(state._h, 0, _lib.ptr(state.last_product)))
        else:
            state.last_data_product = np.empty(A.rows)
            _lib.check(_lib.load().hs_stepper_product(state._h, 0, _lib.ptr(state.last_data_product)))
            if state._n_D > nd_before:
                state.last_solution_product = np.empty(A.cols)
                _lib.check(_lib.load().hs_stepper_product(state._h, 1, _lib.ptr(state.last_solution_product)))
    return state


def step_square(state, A, keep_product=False):
    """hessenberg.py:191-226 on the device: one column of A L_k = L_{k+1} H."""
    return _step(state, A, keep_product, True)


def step_generalized(state, A, keep_products=False):
    """hessenberg.py:329-390 on the device: one column of each basis."""
    return _step(state, A, keep_products, False)


def dump_factorization(state, directory, prefix=""):
    """hessenberg.py:393-406: the factorization pieces as MatrixMarket files."""
    import os

    from .linops import save_array

    def path(name):
        return os.path.join(str(directory), prefix + name)

    save_array(path("L.mm"), state.L_matrix())
    save_array(path("H.mm"), state.H_matrix())
    save_array(path("pivots_t.mm"), np.asarray(state.t, dtype=float))
    if hasattr(state, "W_matrix") and not getattr(state, "square", getattr(state, "_square", False)):
        save_array(path("D.mm"), state.D_matrix())
        save_array(path("W.mm"), state.W_matrix())
        save_array(path("pivots_g.mm"), np.asarray(state.g, dtype=float))
