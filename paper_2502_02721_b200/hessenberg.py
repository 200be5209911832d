"""Pivoting strategy and factorization state of the pivoted Hessenberg
processes (hessenberg.py:48-390 of the reference), as seen from the host.

The processes themselves run on the device inside ``hs_solve``; what comes
back is a :class:`DeviceFactorization` exposing the reference state's fields
(``t``, ``g``, ``k``, ``breakdown``, ``L_cols``, ``D_cols``, ``H_matrix()``,
``W_matrix()``, ``L_matrix()``, ``D_matrix()``).  Basis columns are copied
from the device only when accessed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["PivotStrategy", "TrivialSolution", "DeviceFactorization"]


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

    def __init__(self, result, square, rows, cols):
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

        self.L_cols = _LazyCols(fetch(0, cols), info["n_basis_sol"])
        self.D_cols = None if square else _LazyCols(fetch(1, rows), info["n_basis_data"])
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
