"""Sketch plugin: drop-in for the reference's ``SketchOperator`` /
``make_gaussian_sketch`` / ``sketch_apply`` / ``derive_seed`` (sketch.py:19-123),
plus two device-generated sketch kinds.

* ``make_gaussian_sketch(out_rows, in_rows, seed)`` keeps the reference's
  reproducibility contract bit for bit: ``PCG64(seed).standard_normal`` drawn
  row-major on the host, divided by sqrt(out_rows) (sketch.py:43-53).  This is
  setup, not the loop; the solver uploads the matrix once.
* :class:`GaussianSketch` -- N(0, 1/ell) entries generated on the device from
  a counter-based RNG (Philox-4x32-10 + Box-Muller) every time S is applied;
  never stored.  ``materialize()`` exports the same matrix to the host.
* :class:`SparseSignSketch` -- ``zeta`` nonzeros of +-1/sqrt(zeta) per column
  (rows and signs from Philox), stored by sketch row on the device;
  ``materialize()`` exports it as scipy CSR so the reference can be fed the
  identical S through its ``sketch=`` hook.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import scipy.sparse

from . import _lib

__all__ = [
    "SketchOperator",
    "DeviceSketch",
    "GaussianSketch",
    "SparseSignSketch",
    "make_gaussian_sketch",
    "sketch_apply",
    "derive_seed",
    "device_sketch",
]


@dataclass
class SketchOperator:
    """A realised random embedding of R^in_rows into R^out_rows (sketch.py:29-40).
    ``entries``: ndarray, scipy sparse matrix, or a :class:`DeviceSketch`."""

    out_rows: int
    in_rows: int
    seed: int
    entries: object

    @property
    def shape(self):
        return (self.out_rows, self.in_rows)


def make_gaussian_sketch(out_rows, in_rows, seed):
    """sketch.py:43-53 (host PCG64 draw; identical bits to the reference)."""
    if out_rows < 1 or in_rows < 1:
        raise ValueError("sketch dimensions must be positive")
    gen = np.random.Generator(np.random.PCG64(seed))
    entries = gen.standard_normal((out_rows, in_rows)) / np.sqrt(out_rows)
    return SketchOperator(out_rows, in_rows, int(seed), entries)


def derive_seed(seed, stream):
    """sketch.py:115-123: SeedSequence(seed, spawn_key=(stream,)) child seed."""
    ss = np.random.SeedSequence(int(seed), spawn_key=(int(stream),))
    return int(ss.generate_state(1, dtype=np.uint64)[0])


class DeviceSketch:
    """A sketch living on the device (owns an ``hs_sketch`` handle)."""

    def __init__(self, handle, out_rows, in_rows, seed, ctx):
        self._handle = handle
        self.out_rows = int(out_rows)
        self.in_rows = int(in_rows)
        self.seed = int(seed)
        self.ctx = ctx

    @property
    def handle(self):
        return self._handle

    @property
    def shape(self):
        return (self.out_rows, self.in_rows)

    def apply(self, v, dtype=np.float64):
        v = np.asarray(v)
        code = _lib.HS_F64 if np.dtype(dtype) == np.float64 else _lib.HS_F32
        if v.ndim == 2:
            # entries @ Q for a block of columns (sketch.py:108): one generator
            # pass per 8 columns for the Gaussian kind, each column bit-identical
            # to a single apply
            if v.shape[0] != self.in_rows:
                raise ValueError(f"sketch expects {self.in_rows} rows, got shape {v.shape}")
            vt = np.ascontiguousarray(v.T, dtype=dtype)
            out = np.empty((v.shape[1], self.out_rows))
            _lib.check(_lib.load().hs_sketch_apply_many(self._handle, code, int(v.shape[1]), _lib.ptr(vt),
                                                        _lib.ptr(out)))
            return np.ascontiguousarray(out.T)
        v = np.ascontiguousarray(v, dtype=dtype)
        if v.shape != (self.in_rows,):
            raise ValueError(f"sketch expects a vector of length {self.in_rows}, got shape {v.shape}")
        out = np.empty(self.out_rows)
        _lib.check(_lib.load().hs_sketch_apply(self._handle, code, _lib.ptr(v), _lib.ptr(out)))
        return out

    def __matmul__(self, v):
        return self.apply(v)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                _lib.load().hs_sketch_destroy(h)
            except Exception:
                pass
            self._handle = None


class GaussianSketch(DeviceSketch):
    """N(0, 1/out_rows) entries regenerated on the device at every application."""

    def __init__(self, out_rows, in_rows, seed=0, device=None):
        ctx = _lib.context(device)
        h = _lib.c_vp()
        _lib.check(_lib.load().hs_sketch_create(ctx.handle, _lib.HS_SKETCH_GAUSSIAN, int(out_rows), int(in_rows),
                                                int(seed) & 0xFFFFFFFFFFFFFFFF, 0, None, ctypes.byref(h)))
        super().__init__(h, out_rows, in_rows, seed, ctx)

    def materialize(self):
        out = np.empty((self.out_rows, self.in_rows))
        _lib.check(_lib.load().hs_sketch_materialize(self._handle, _lib.ptr(out)))
        return out


class SparseSignSketch(DeviceSketch):
    """``zeta`` entries of +-1/sqrt(zeta) per column, distinct rows."""

    def __init__(self, out_rows, in_rows, seed=0, zeta=8, device=None):
        ctx = _lib.context(device)
        h = _lib.c_vp()
        _lib.check(_lib.load().hs_sketch_create(ctx.handle, _lib.HS_SKETCH_SPARSE_SIGN, int(out_rows), int(in_rows),
                                                int(seed) & 0xFFFFFFFFFFFFFFFF, int(zeta), None, ctypes.byref(h)))
        self.zeta = int(zeta)
        super().__init__(h, out_rows, in_rows, seed, ctx)

    def materialize(self):
        nnz = _lib.c_i64()
        _lib.check(_lib.load().hs_sketch_nnz(self._handle, ctypes.byref(nnz)))
        indptr = np.empty(self.out_rows + 1, dtype=np.int64)
        indices = np.empty(nnz.value, dtype=np.int32)
        data = np.empty(nnz.value)
        _lib.check(_lib.load().hs_sketch_export_csr(self._handle, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(data)))
        return scipy.sparse.csr_matrix((data, indices, indptr), shape=(self.out_rows, self.in_rows))


class _ExplicitSketch(DeviceSketch):
    """An explicit S (dense ndarray or scipy sparse) uploaded once."""

    def __init__(self, entries, seed=0, device=None):
        ctx = _lib.context(device)
        h = _lib.c_vp()
        lib = _lib.load()
        if scipy.sparse.issparse(entries):
            M = scipy.sparse.csr_matrix(entries, dtype=np.float64)
            M.sort_indices()
            indptr = np.ascontiguousarray(M.indptr, dtype=np.int64)
            indices = np.ascontiguousarray(M.indices, dtype=np.int32)
            data = np.ascontiguousarray(M.data, dtype=np.float64)
            _lib.check(lib.hs_sketch_create_csr(ctx.handle, M.shape[0], M.shape[1], int(M.nnz), _lib.ptr(indptr),
                                                _lib.ptr(indices), _lib.ptr(data), ctypes.byref(h)))
            shape = M.shape
        else:
            E = np.ascontiguousarray(entries, dtype=np.float64)
            if E.ndim != 2:
                raise ValueError("sketch entries must be 2-D")
            _lib.check(lib.hs_sketch_create(ctx.handle, _lib.HS_SKETCH_DENSE, E.shape[0], E.shape[1], 0, 0,
                                            _lib.ptr(E), ctypes.byref(h)))
            shape = E.shape
        super().__init__(h, shape[0], shape[1], seed, ctx)


def device_sketch(sk):
    """A :class:`DeviceSketch` for a ``SketchOperator`` (or a DeviceSketch)."""
    if isinstance(sk, DeviceSketch):
        return sk
    entries = getattr(sk, "entries", None)
    if isinstance(entries, DeviceSketch):
        return entries
    if entries is None:
        raise TypeError("sketch has no entries")
    return _ExplicitSketch(entries, getattr(sk, "seed", 0))


def sketch_apply(S, v, counters=None):
    """sketch.py:56-65 on the device: S v plus one sketch count."""
    v = np.asarray(v, dtype=float)
    if v.shape != (S.in_rows,):
        raise ValueError(f"sketch expects a vector of length {S.in_rows}, got shape {v.shape}")
    if counters is not None:
        counters.sketch_apply_count += 1
    return device_sketch(S).apply(v)
