"""Operator plugin: drop-in for the reference's ``LinearOperator``
(linops.py:53-149) whose forward / transpose applications run on the B200.

Device-backed operators (each owns an ``hs_op`` handle, C ABI
``include/hessketch_b200.h``):

* :class:`DenseOperator`   -- ``from_matrix(ndarray)``        (linops.py:142-145)
* :class:`CsrOperator`     -- ``from_matrix(scipy sparse)``   (linops.py:137-141)
* :class:`PsfOperator`     -- ``make_deblur`` closures         (problems.py:257-267)
* :class:`TomographyOperator` -- ``make_tomography`` matrix built on device
  (problems.py:311-331)

``LinearOperator(rows, cols, forward, transpose)`` with arbitrary Python
callables is accepted for API compatibility (``apply`` calls the user's
callables), but the solvers refuse it with ``TypeError``: this package has no
CPU path for the hot loop.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse

from . import _lib

__all__ = [
    "OpCounters",
    "LinearOperator",
    "DeviceOperator",
    "DenseOperator",
    "CsrOperator",
    "PsfOperator",
    "TomographyOperator",
    "to_device_operator",
    "spectral_condition_number",
    "save_array",
    "load_array",
    "load_operator",
]


@dataclass
class OpCounters:
    """linops.py:53-68."""

    matvec_count: int = 0
    transpose_matvec_count: int = 0
    dot_product_count: int = 0
    sketch_apply_count: int = 0

    def snapshot(self):
        return (
            self.matvec_count,
            self.transpose_matvec_count,
            self.dot_product_count,
            self.sketch_apply_count,
        )


class LinearOperator:
    """A real m x n linear map accessed through its action on vectors
    (linops.py:71-149: same fields, same validation and counting)."""

    def __init__(self, rows, cols, forward=None, transpose=None, counters=None):
        if rows < 1 or cols < 1:
            raise ValueError("operator dimensions must be positive")
        self.rows = int(rows)
        self.cols = int(cols)
        self.forward = forward
        self.transpose = transpose
        self.counters = counters if counters is not None else OpCounters()

    @property
    def shape(self):
        return (self.rows, self.cols)

    @property
    def is_square(self):
        return self.rows == self.cols

    def apply(self, x):
        """Return A @ x and count one forward application (linops.py:107-115)."""
        x = np.asarray(x, dtype=float)
        if x.shape != (self.cols,):
            raise ValueError(f"operator expects a vector of length {self.cols}, got shape {x.shape}")
        self.counters.matvec_count += 1
        return np.asarray(self.forward(x), dtype=float)

    def apply_transpose(self, y):
        """Return A.T @ y and count one transpose application (linops.py:117-125)."""
        y = np.asarray(y, dtype=float)
        if y.shape != (self.rows,):
            raise ValueError(
                f"operator transpose expects a vector of length {self.rows}, got shape {y.shape}"
            )
        self.counters.transpose_matvec_count += 1
        return np.asarray(self.transpose(y), dtype=float)

    def with_fresh_counters(self):
        """A view of the same map with zeroed counters (linops.py:127-133)."""
        return LinearOperator(self.rows, self.cols, self.forward, self.transpose)

    @classmethod
    def from_matrix(cls, M):
        """Wrap a dense array or scipy sparse matrix as a device operator."""
        if scipy.sparse.issparse(M):
            return CsrOperator(M)
        M = np.asarray(M)
        if M.ndim != 2:
            raise ValueError("expected a 2-D matrix")
        return DenseOperator(M)

    @classmethod
    def identity(cls, n):
        return CsrOperator(scipy.sparse.identity(int(n), format="csr", dtype=np.float64))


class DeviceOperator(LinearOperator):
    """Base of the operators whose applications run on the device."""

    kind = "device"

    def __init__(self, rows, cols, handle, value_dtype, ctx, counters=None, owner=None):
        super().__init__(rows, cols, self._fwd, self._tr, counters)
        self._handle = handle
        self.value_dtype = np.dtype(value_dtype)
        self.ctx = ctx
        self._owner = owner  # the operator that owns the native handle (views share it)

    @property
    def handle(self):
        return self._handle

    def _apply(self, v, transpose, work=np.float64):
        work = np.dtype(work)
        n_in = self.rows if transpose else self.cols
        n_out = self.cols if transpose else self.rows
        v = np.ascontiguousarray(v, dtype=work)
        if v.shape != (n_in,):
            raise ValueError(f"expected a vector of length {n_in}")
        out = np.empty(n_out, dtype=work)
        code = _lib.HS_F64 if work == np.float64 else _lib.HS_F32
        _lib.check(_lib.load().hs_op_apply(self._handle, 1 if transpose else 0, code, _lib.ptr(v), _lib.ptr(out)))
        return out

    def _fwd(self, x):
        return self._apply(x, False)

    def _tr(self, y):
        return self._apply(y, True)

    def matvec(self, x, dtype=np.float64):
        """Uncounted device A x in the given working precision."""
        return self._apply(x, False, dtype)

    def rmatvec(self, y, dtype=np.float64):
        """Uncounted device A^T y in the given working precision."""
        return self._apply(y, True, dtype)

    def with_fresh_counters(self):
        view = object.__new__(type(self))
        view.__dict__.update(self.__dict__)
        view.counters = OpCounters()
        view.forward, view.transpose = view._fwd, view._tr
        view._owner = self._owner or self
        return view

    def info(self):
        m, n, nnz, nnzt = _lib.c_i64(), _lib.c_i64(), _lib.c_i64(), _lib.c_i64()
        _lib.check(_lib.load().hs_op_info(self._handle, ctypes.byref(m), ctypes.byref(n), ctypes.byref(nnz), ctypes.byref(nnzt)))
        return {"rows": m.value, "cols": n.value, "nnz": nnz.value, "nnz_t": nnzt.value}

    def storage(self, transpose=False):
        """How the SELL copy of A (or A^T) is stored on the device: slices, entry
        slots, the slices / slots on compact step codes, index bytes per nonzero."""
        sl, so, cs, co = _lib.c_i64(), _lib.c_i64(), _lib.c_i64(), _lib.c_i64()
        ib = ctypes.c_double()
        _lib.check(_lib.load().hs_op_storage(self._handle, 1 if transpose else 0, ctypes.byref(sl), ctypes.byref(so),
                                             ctypes.byref(cs), ctypes.byref(co), ctypes.byref(ib)))
        return {"slices": sl.value, "slots": so.value, "code_slices": cs.value, "code_slots": co.value,
                "index_bytes_per_nnz": ib.value}

    def __del__(self):
        if getattr(self, "_owner", None) is None and getattr(self, "_handle", None) is not None:
            try:
                _lib.load().hs_op_destroy(self._handle)
            except Exception:
                pass
            self._handle = None


def _value_code(dt):
    dt = np.dtype(dt)
    if dt == np.float64:
        return _lib.HS_F64
    if dt == np.float32:
        return _lib.HS_F32
    raise TypeError(f"operator values must be float64 or float32, got {dt}")


class DenseOperator(DeviceOperator):
    """Dense m x n matrix (row-major input), values fp64 or fp32."""

    kind = "dense"

    def __init__(self, M, dtype=None, device=None):
        M = np.asarray(M)
        if M.ndim != 2:
            raise ValueError("expected a 2-D matrix")
        dt = np.dtype(dtype) if dtype is not None else (np.float32 if M.dtype == np.float32 else np.float64)
        M = np.ascontiguousarray(M, dtype=dt)
        ctx = _lib.context(device)
        h = _lib.c_vp()
        _lib.check(_lib.load().hs_op_dense_create(ctx.handle, M.shape[0], M.shape[1], _lib.ptr(M), _value_code(dt), ctypes.byref(h)))
        super().__init__(M.shape[0], M.shape[1], h, dt, ctx)


class CsrOperator(DeviceOperator):
    """Sparse operator; A and A^T are kept as row-sorted CSR on the device
    (scipy's ``M`` and ``M.T.tocsr()``, linops.py:137-141)."""

    kind = "csr"

    def __init__(self, M, dtype=None, device=None):
        M = scipy.sparse.csr_matrix(M)
        if not M.has_sorted_indices:
            M = M.sorted_indices()
        M.sum_duplicates()
        dt = np.dtype(dtype) if dtype is not None else (np.float32 if M.dtype == np.float32 else np.float64)
        indptr = np.ascontiguousarray(M.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(M.indices, dtype=np.int32)
        data = np.ascontiguousarray(M.data, dtype=dt)
        ctx = _lib.context(device)
        h = _lib.c_vp()
        _lib.check(_lib.load().hs_op_csr_create(
            ctx.handle, M.shape[0], M.shape[1], int(M.nnz), _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(data),
            _value_code(dt), ctypes.byref(h)))
        super().__init__(M.shape[0], M.shape[1], h, dt, ctx)

    def export(self, transpose=False):
        """Device CSR (A or A^T) back to host as scipy CSR (float64 data)."""
        inf = self.info()
        rows = inf["cols"] if transpose else inf["rows"]
        cols = inf["rows"] if transpose else inf["cols"]
        nnz = inf["nnz_t"] if transpose else inf["nnz"]
        indptr = np.empty(rows + 1, dtype=np.int64)
        indices = np.empty(max(nnz, 1), dtype=np.int32)
        data = np.empty(max(nnz, 1), dtype=np.float64)
        _lib.check(_lib.load().hs_op_export_csr(self._handle, 1 if transpose else 0, _lib.ptr(indptr), _lib.ptr(indices), _lib.ptr(data)))
        return scipy.sparse.csr_matrix((data[:nnz], indices[:nnz], indptr), shape=(rows, cols))


class TomographyOperator(CsrOperator):
    """Parallel-beam exact-chord projector built on the device.

    Rows ``a * n_bins + j`` (angle a, detector j), columns ``r * grid + c``;
    the angle table and detector offsets are computed here exactly as the
    reference computes them (problems.py:317-322), so with ``n_bins == grid``
    the device matrix equals ``problems.tomography_matrix(grid, n_angles)``
    bit for bit (``dtype=float64``), or its float32 rounding."""

    kind = "tomography"

    def __init__(self, grid, n_angles, n_bins=None, dtype=np.float32, device=None):
        grid, n_angles = int(grid), int(n_angles)
        n_bins = grid if n_bins is None else int(n_bins)
        cos_t = np.array([math.cos(math.pi * a / n_angles) for a in range(n_angles)])
        sin_t = np.array([math.sin(math.pi * a / n_angles) for a in range(n_angles)])
        offsets = np.array([j + 0.5 - n_bins / 2.0 for j in range(n_bins)])
        dt = np.dtype(dtype)
        ctx = _lib.context(device)
        h = _lib.c_vp()
        _lib.check(_lib.load().hs_op_tomo_create(
            ctx.handle, grid, n_angles, n_bins, _lib.ptr(cos_t), _lib.ptr(sin_t), _lib.ptr(offsets),
            _value_code(dt), ctypes.byref(h)))
        self.grid, self.n_angles, self.n_bins = grid, n_angles, n_bins
        DeviceOperator.__init__(self, n_angles * n_bins, grid * grid, h, dt, ctx)


class PsfOperator(DeviceOperator):
    """Zero-boundary 'same' 2-D convolution with an odd-sided PSF; the
    transpose is correlation (problems.py:257-267).  Taps are summed in a fixed
    order (oracle/tomo_oracle.py:psf_stencil)."""

    kind = "psf"

    def __init__(self, shape, psf, dtype=np.float64, device=None):
        if np.isscalar(shape):
            shape = (int(shape), int(shape))
        H, W = int(shape[0]), int(shape[1])
        K = np.ascontiguousarray(psf, dtype=np.float64)
        if K.ndim != 2 or K.shape[0] % 2 == 0 or K.shape[1] % 2 == 0:
            raise ValueError("psf must be a 2-D kernel with odd side lengths")
        if K.shape[0] >= H or K.shape[1] >= W:
            raise ValueError("psf support must be smaller than the image")
        dt = np.dtype(dtype)
        ctx = _lib.context(device)
        h = _lib.c_vp()
        _lib.check(_lib.load().hs_op_psf_create(ctx.handle, H, W, K.shape[0], K.shape[1], _lib.ptr(K), _value_code(dt), ctypes.byref(h)))
        self.image_shape = (H, W)
        self.psf = K
        super().__init__(H * W, H * W, h, dt, ctx)


def to_device_operator(A):
    """Return a device operator for ``A`` or raise ``TypeError``.

    Accepts this package's device operators, and the reference's own
    ``LinearOperator.from_matrix`` objects (the wrapped ndarray / scipy matrix
    is recovered from the closure, linops.py:140-145)."""
    if isinstance(A, DeviceOperator):
        return A
    fwd = getattr(A, "forward", None)
    cells = getattr(fwd, "__closure__", None) or ()
    for cell in cells:
        try:
            obj = cell.cell_contents
        except ValueError:
            continue
        if scipy.sparse.issparse(obj) and obj.shape == (A.rows, A.cols):
            return CsrOperator(obj)
        if isinstance(obj, np.ndarray) and obj.shape == (A.rows, A.cols):
            return DenseOperator(obj)
    raise TypeError(
        "operator has no device implementation (Python callables are not run on the GPU); "
        "use DenseOperator / CsrOperator / PsfOperator / TomographyOperator or from_matrix"
    )


# ---------------------------------------------------------------------------
# exchange formats (linops.py:235-282): MatrixMarket files and the condition
# number the reference's diagnostics report.  Host-side I/O around the device
# path; ``load_operator`` returns a device operator.


def spectral_condition_number(M):
    """sigma_max / sigma_min by SVD (linops.py:235-247); inf when sigma_min
    underflows below 1e-300; ValueError for an empty or all-zero matrix."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2 or M.size == 0:
        raise ValueError("expected a nonempty 2-D matrix")
    sv = np.linalg.svd(M, compute_uv=False)
    if sv[0] == 0.0:
        raise ValueError("condition number of the zero matrix is undefined")
    return np.inf if sv[-1] < 1e-300 else float(sv[0] / sv[-1])


def save_array(path, arr):
    """MatrixMarket array file of a vector (one column) or matrix
    (linops.py:249-260); the path is used verbatim."""
    import scipy.io

    a = np.asarray(arr, dtype=float)
    a = a[:, None] if a.ndim == 1 else a
    with open(path, "wb") as fh:
        scipy.io.mmwrite(fh, a)


def load_array(path):
    """Dense array from a MatrixMarket file; single columns come back 1-D
    (linops.py:262-271)."""
    import scipy.io

    with open(path, "rb") as fh:
        a = scipy.io.mmread(fh)
    a = np.asarray(a.toarray() if scipy.sparse.issparse(a) else a, dtype=float)
    return a[:, 0].copy() if (a.ndim == 2 and a.shape[1] == 1) else a


def load_operator(path):
    """Device operator from a MatrixMarket file (linops.py:274-282):
    coordinate files -> :class:`CsrOperator`, array files -> :class:`DenseOperator`."""
    import scipy.io

    with open(path, "rb") as fh:
        M = scipy.io.mmread(fh)
    return LinearOperator.from_matrix(M)


# ---------------------------------------------------------------------------
# projected least squares (linops.py:34-50, 168-229) on the device


RANK_TOL = 1e-14


class RankDeficiencyError(np.linalg.LinAlgError):
    """linops.py:39-50: raised with the detected numerical rank."""

    def __init__(self, message, rank):
        super().__init__(message)
        self.rank = rank


def dense_qr_ls(M, rhs):
    """linops.py:168-207 on the device: min_y |M y - rhs| for l >= k, by the
    loop's incremental CGS2 QR (hs_qr.cuh).  Raises RankDeficiencyError when a
    column fails the RANK_TOL gate (the solvers then use the minimum-norm
    solution, which the device forms from the same factorisation)."""
    M = np.asarray(M, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    if M.ndim != 2:
        raise ValueError("M must be 2-D")
    l, k = M.shape
    if l < k:
        raise ValueError(f"need at least as many rows as columns, got {M.shape}")
    if rhs.shape != (l,):
        raise ValueError(f"rhs must have length {l}, got shape {rhs.shape}")
    if k == 0:
        return np.empty(0)
    Mc = np.asfortranarray(M)
    rhs = np.ascontiguousarray(rhs)
    y = np.empty(k)
    rank = _lib.c_i32()
    _lib.check(_lib.load().hs_projected_ls(_lib.context().handle, l, k, ctypes.c_void_p(Mc.ctypes.data), _lib.ptr(rhs),
                                           _lib.ptr(y), ctypes.byref(rank)))
    if rank.value < k:
        raise RankDeficiencyError(f"matrix is numerically rank deficient (rank {rank.value} of {k})", rank.value)
    return y


def stacked_tikhonov_ls(M, N, rhs, lam):
    """linops.py:210-229: min |M y - rhs|^2 + lam^2 |N y|^2 as the stacked
    system [M; lam N] y ~ [rhs; 0]; lam == 0 takes exactly dense_qr_ls."""
    if lam < 0:
        raise ValueError("lam must be nonnegative")
    if lam == 0.0:
        return dense_qr_ls(M, rhs)
    M = np.asarray(M, dtype=float)
    N = np.asarray(N, dtype=float)
    rhs = np.asarray(rhs, dtype=float)
    if N.shape[1] != M.shape[1]:
        raise ValueError("M and N must have the same number of columns")
    return dense_qr_ls(np.vstack([M, lam * N]), np.concatenate([rhs, np.zeros(N.shape[0])]))
