"""ctypes binding of the C ABI in include/hessketch_b200.h.

The shared library is built in-tree (``paper_2502_02721_b200/_build/libhessketch_b200.so``,
see ``build.py``).  There is no fallback: if the library is missing, or no
CUDA device is usable, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libhessketch_b200.so")

HS_OK, HS_ERR_VALUE, HS_ERR_RUNTIME, HS_ERR_CUDA, HS_ERR_NOTIMPL, HS_ERR_TYPE, HS_ERR_COMM = range(7)
HS_F64, HS_F32, HS_BF16 = 0, 1, 2
HS_SKETCH_DENSE, HS_SKETCH_GAUSSIAN, HS_SKETCH_SPARSE_SIGN, HS_SKETCH_CSR = 0, 1, 2, 3
TERMINATIONS = {0: "maxiter", 1: "breakdown", 2: "trivial"}

DTYPE_CODES = {"float64": HS_F64, "float32": HS_F32, "bfloat16": HS_BF16}

c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)
P_dbl = ctypes.POINTER(ctypes.c_double)


class HsConfig(ctypes.Structure):
    """hs_config (include/hessketch_b200.h)."""

    _fields_ = [
        ("maxiter", ctypes.c_int32),
        ("square", ctypes.c_int32),
        ("sketch_basis", ctypes.c_int32),
        ("work_dtype", ctypes.c_int32),
        ("basis_dtype", ctypes.c_int32),
        ("record_x", ctypes.c_int32),
        ("lam", ctypes.c_double),
        ("sketched", ctypes.c_int32),
        ("pivot_sample", ctypes.c_int32),
        ("pivot_positions", ctypes.c_void_p),
        ("diagnostics", ctypes.c_int32),
        ("printed_f", ctypes.c_int32),
    ]


# (name, restype, argtypes); every function returns an hs_status int
_SIGNATURES = [
    ("hs_last_error", ctypes.c_char_p, []),
    ("hs_version", ctypes.c_char_p, []),
    ("hs_launch_count", ctypes.c_ulonglong, []),
    ("hs_guard_violations", ctypes.c_ulonglong, []),
    ("hs_ctx_create", c_i32, [ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("hs_ctx_destroy", c_i32, [c_vp]),
    ("hs_ctx_synchronize", c_i32, [c_vp]),
    ("hs_ctx_set_profiling", c_i32, [c_vp, ctypes.c_int]),
    ("hs_ctx_reset_stats", c_i32, [c_vp]),
    ("hs_ctx_kernel_stats", c_i32, [c_vp, ctypes.c_char_p, P_i64, P_dbl, P_dbl]),
    ("hs_ctx_kernel_names", c_i32, [c_vp, ctypes.c_char_p, c_i64]),
    ("hs_comm_get_unique_id", c_i32, [c_vp]),
    ("hs_comm_init", c_i32, [c_vp, ctypes.c_int, ctypes.c_int, c_vp]),
    ("hs_nccl_selftest", c_i32, [c_vp]),
    ("hs_comm_info", c_i32, [c_vp, P_i32, P_i32]),
    ("hs_comm_init_local", c_i32, [ctypes.POINTER(c_vp), ctypes.c_int]),
    ("hs_comm_abort", c_i32, [c_vp]),
    ("hs_ctx_force_sharding", c_i32, [c_vp, ctypes.c_int]),
    ("hs_op_shard_info", c_i32, [c_vp, P_i64, P_i64, P_i64, P_i64, P_i64, P_i64]),
    ("hs_op_dense_create", c_i32, [c_vp, c_i64, c_i64, c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("hs_op_csr_create", c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("hs_op_psf_create", c_i32, [c_vp, c_i64, c_i64, c_i32, c_i32, c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("hs_op_tomo_create", c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, ctypes.c_int, ctypes.POINTER(c_vp)]),
    ("hs_op_info", c_i32, [c_vp, P_i64, P_i64, P_i64, P_i64]),
    ("hs_op_storage", c_i32, [c_vp, c_i32, P_i64, P_i64, P_i64, P_i64, ctypes.POINTER(ctypes.c_double)]),
    ("hs_op_apply", c_i32, [c_vp, ctypes.c_int, ctypes.c_int, c_vp, c_vp]),
    ("hs_op_export_csr", c_i32, [c_vp, ctypes.c_int, c_vp, c_vp, c_vp]),
    ("hs_op_destroy", c_i32, [c_vp]),
    ("hs_sketch_create", c_i32, [c_vp, ctypes.c_int, c_i64, c_i64, ctypes.c_uint64, c_i32, c_vp, ctypes.POINTER(c_vp)]),
    ("hs_sketch_create_csr", c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("hs_sketch_apply", c_i32, [c_vp, ctypes.c_int, c_vp, c_vp]),
    ("hs_sketch_apply_many", c_i32, [c_vp, ctypes.c_int, c_i32, c_vp, c_vp]),
    ("hs_sketch_materialize", c_i32, [c_vp, c_vp]),
    ("hs_sketch_nnz", c_i32, [c_vp, P_i64]),
    ("hs_sketch_export_csr", c_i32, [c_vp, c_vp, c_vp, c_vp]),
    ("hs_sketch_destroy", c_i32, [c_vp]),
    ("hs_solve", c_i32, [c_vp, c_vp, ctypes.POINTER(HsConfig), c_vp, c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("hs_solve_krylov", c_i32, [c_vp, c_vp, ctypes.POINTER(HsConfig), c_i32, c_vp, c_vp, c_vp, ctypes.POINTER(c_vp)]),
    ("hs_result_info", c_i32, [c_vp, P_i32, P_i32, P_i32, P_i32, P_i32, P_i32]),
    ("hs_result_x", c_i32, [c_vp, c_vp]),
    ("hs_result_resnorm", c_i32, [c_vp, c_vp]),
    ("hs_result_diagnostics", c_i32, [c_vp, c_vp, c_vp, c_vp]),
    ("hs_result_trace", c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    ("hs_result_pivots", c_i32, [c_vp, c_vp, c_vp]),
    ("hs_result_hessenberg", c_i32, [c_vp, c_vp, c_vp]),
    ("hs_result_basis", c_i32, [c_vp, ctypes.c_int, c_i32, c_vp]),
    ("hs_result_projected", c_i32, [c_vp, c_vp, c_vp, c_vp]),
    ("hs_result_loop_ms", c_i32, [c_vp, P_dbl]),
    ("hs_result_destroy", c_i32, [c_vp]),
    ("hs_stepper_create", c_i32, [c_vp, c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp, P_i32,
                                  ctypes.POINTER(c_vp)]),
    ("hs_stepper_step", c_i32, [c_vp, c_i32, c_vp]),
    ("hs_stepper_info", c_i32, [c_vp, P_i32, P_i32, P_i32, P_i32, P_i32, P_dbl, P_dbl]),
    ("hs_stepper_hessenberg", c_i32, [c_vp, c_vp, c_vp]),
    ("hs_stepper_pivots", c_i32, [c_vp, c_vp, c_vp]),
    ("hs_stepper_basis", c_i32, [c_vp, c_i32, c_i32, c_vp]),
    ("hs_stepper_product", c_i32, [c_vp, c_i32, c_vp]),
    ("hs_stepper_r0", c_i32, [c_vp, c_vp]),
    ("hs_stepper_destroy", c_i32, [c_vp]),
    ("hs_pivot_select", c_i32, [c_vp, c_i64, c_vp, c_i64, c_vp, P_i64, P_dbl]),
    ("hs_projected_ls", c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, P_i32]),
]

EXPORTED = [name for name, _, _ in _SIGNATURES]

_lib = None
_lock = threading.Lock()


class HsLibraryError(RuntimeError):
    """The native library is missing or failed to load."""


def load(path=None):
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise HsLibraryError(
                f"native library {p} not built; run paper_2502_02721_b200.build.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(p)
        for name, res, args in _SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(status):
    """Map an hs_status to the reference's exception types."""
    if status == HS_OK:
        return
    msg = load().hs_last_error().decode("utf-8", "replace")
    if status == HS_ERR_VALUE:
        raise ValueError(msg)
    if status == HS_ERR_NOTIMPL:
        raise NotImplementedError(msg)
    if status == HS_ERR_TYPE:
        raise TypeError(msg)
    raise RuntimeError(f"hessketch_b200 error {status}: {msg}")


def ptr(a):
    """ctypes pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return ctypes.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# per-process context on the current CUDA device


class Context:
    def __init__(self, device=0):
        lib = load()
        h = c_vp()
        check(lib.hs_ctx_create(int(device), ctypes.byref(h)))
        self.handle = h
        self.device = int(device)
        self._lib = lib

    def synchronize(self):
        check(self._lib.hs_ctx_synchronize(self.handle))

    def close(self):
        """Destroy the context (objects created on it keep their buffers valid)."""
        h, self.handle = self.handle, None
        if h is not None:
            check(self._lib.hs_ctx_destroy(h))

    def set_profiling(self, on):
        check(self._lib.hs_ctx_set_profiling(self.handle, 1 if on else 0))

    def reset_stats(self):
        check(self._lib.hs_ctx_reset_stats(self.handle))

    def kernel_stats(self):
        buf = ctypes.create_string_buffer(1 << 16)
        check(self._lib.hs_ctx_kernel_names(self.handle, buf, len(buf)))
        out = {}
        for name in buf.value.decode().split("\n"):
            if not name:
                continue
            n, ms, by = c_i64(), c_dbl(), c_dbl()
            check(self._lib.hs_ctx_kernel_stats(self.handle, name.encode(), ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by)))
            out[name] = {"launches": n.value, "ms": ms.value, "bytes": by.value}
        return out


_ctx = {}
_tls = threading.local()


class use_context:
    """``with use_context(ctx):`` -- objects created and solves run on this
    thread use ``ctx`` instead of the process-wide context (one host thread per
    in-process rank, :func:`paper_2502_02721_b200.dist.local_group`)."""

    def __init__(self, ctx):
        self.ctx = ctx

    def __enter__(self):
        self.prev = getattr(_tls, "ctx", None)
        _tls.ctx = self.ctx
        return self.ctx

    def __exit__(self, *exc):
        _tls.ctx = self.prev


def context(device=None):
    """The context of this thread (:class:`use_context`), else the
    process-wide context for ``device`` (default: LOCAL_RANK or 0)."""
    over = getattr(_tls, "ctx", None)
    if over is not None and (device is None or int(device) == over.device):
        return over
    if device is None:
        device = int(os.environ.get("HS_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _lock:
        c = _ctx.get(device)
    if c is None:
        c = Context(device)
        with _lock:
            _ctx[device] = c
    return c


def as_f64(a, n=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if n is not None and a.shape != (n,):
        raise ValueError(f"expected a vector of length {n}, got shape {a.shape}")
    return a
