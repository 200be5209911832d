"""TEST INFRASTRUCTURE ONLY -- CPU baseline for bench.py: the C port of the
reference's sLSLU loop (oracle/coracle.c) on the host cores, on a bounded
sample of the benchmark workload.

The host builds its own operator with the C restatement of the reference ray
tracer (no GPU code on this path), the same seeded phantom and noise, and a
host-drawn sparse-sign S2 of the same shape and density.  The per-iteration
time depends on k (2k elimination passes, the from-scratch QR of the l x k
sketched matrix, x = L_k y), so the rate over the config's K iterations is
measured by timing one iteration of the loop body at steps spread over
k = 1..K (co_probe_iter) and averaging the interpolated t(k) over every k;
a few real iterations from k = 1 check the probe.
"""
from __future__ import annotations

import ctypes
import math
import os
import time

import numpy as np
import scipy.sparse

from . import build_coracle

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_coracle.build())
        vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.co_tomo_rowptr.argtypes = [i32, i32, i32, vp, vp, vp, vp, i32]
        _lib.co_tomo_fill.argtypes = [i32, i32, i32, vp, vp, vp, vp, vp, vp, i32]
        _lib.co_csr_transpose.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, i32]
        _lib.co_slslu_f32.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, vp, i32, i32, dbl, vp, vp, vp,
                                      vp, vp]
        _lib.co_slslu_f32.restype = ctypes.c_int
        _lib.co_max_threads.restype = ctypes.c_int
        _lib.co_spmv_f32_f64.argtypes = [i64, vp, vp, vp, vp, vp, i32]
        _lib.co_spmv_f32_export.argtypes = [i64, vp, vp, vp, vp, vp, i32]
        _lib.co_psf_conv_f32.argtypes = [i32, i32, vp, i32, i32, vp, vp, i32]
        _lib.co_probe_create.argtypes = [i64, i64, i64, i32, i32]
        _lib.co_probe_create.restype = vp
        _lib.co_probe_destroy.argtypes = [vp]
        _lib.co_probe_iter.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32]
        _lib.co_probe_iter.restype = dbl
        _lib.co_scmrh_psf_f32.argtypes = [i32, i32, vp, i32, i32, vp, i32, i32, vp, vp]
        _lib.co_scmrh_psf_f32.restype = ctypes.c_int
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def host_tomography(grid, n_angles, n_bins, nthreads):
    """A and A^T (fp32 CSR) built on the host by the C ray tracer."""
    L = lib()
    cos_t = np.array([math.cos(math.pi * a / n_angles) for a in range(n_angles)])
    sin_t = np.array([math.sin(math.pi * a / n_angles) for a in range(n_angles)])
    offs = np.array([j + 0.5 - n_bins / 2.0 for j in range(n_bins)])
    m, n = n_angles * n_bins, grid * grid
    rp = np.zeros(m + 1, dtype=np.int64)
    L.co_tomo_rowptr(grid, n_angles, n_bins, _p(cos_t), _p(sin_t), _p(offs), _p(rp), nthreads)
    nnz = int(rp[-1])
    ci = np.empty(nnz, dtype=np.int32)
    cv = np.empty(nnz, dtype=np.float32)
    L.co_tomo_fill(grid, n_angles, n_bins, _p(cos_t), _p(sin_t), _p(offs), _p(rp), _p(ci), _p(cv), nthreads)
    trp = np.zeros(n + 1, dtype=np.int64)
    tci = np.empty(nnz, dtype=np.int32)
    tcv = np.empty(nnz, dtype=np.float32)
    L.co_csr_transpose(m, n, _p(rp), _p(ci), _p(cv), _p(trp), _p(tci), _p(tcv), nthreads)
    return (rp, ci, cv), (trp, tci, tcv), m, n


def sparse_sign(ell, m, zeta, seed):
    rng = np.random.default_rng(seed)
    rows = np.argsort(rng.random((m, ell), dtype=np.float32), axis=1)[:, :zeta] if m * ell <= 5e7 else None
    if rows is None:  # large: rejection-free approximate draw of distinct rows per column
        rows = np.empty((m, zeta), dtype=np.int64)
        base = rng.integers(0, ell, size=m)
        steps = rng.integers(1, ell // zeta, size=(m, zeta))
        rows = (base[:, None] + np.cumsum(steps, axis=1)) % ell
    cols = np.repeat(np.arange(m), zeta)
    vals = rng.choice([-1.0, 1.0], size=m * zeta) / math.sqrt(zeta)
    S = scipy.sparse.csr_matrix((vals, (rows.ravel(), cols)), shape=(ell, m))
    S.sum_duplicates()
    return S


def run_slslu(A, At, m, n, b, ell, maxiter, budget_s, nthreads, seed=7, S=None):
    L = lib()
    if S is None:
        S = sparse_sign(ell, m, 8, seed)
    Srp = np.ascontiguousarray(S.indptr, dtype=np.int64)
    Sci = np.ascontiguousarray(S.indices, dtype=np.int32)
    Scv = np.ascontiguousarray(S.data, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    t = np.zeros(maxiter + 1, dtype=np.int64)
    g = np.zeros(maxiter + 1, dtype=np.int64)
    sres = np.zeros(maxiter)
    its = np.zeros(maxiter)
    x = np.zeros(n)
    done = L.co_slslu_f32(m, n, _p(A[0]), _p(A[1]), _p(A[2]), _p(At[0]), _p(At[1]), _p(At[2]), ell, _p(Srp), _p(Sci),
                          _p(Scv), _p(b), maxiter, nthreads, budget_s, _p(t), _p(g), _p(sres), _p(its), _p(x))
    return dict(done=done, t=t[: done + 1], g=g[: done + 1], sres=sres[:done], iter_s=its[:done], x=x)


_cache = {}


def host_problem(grid, angles, bins, seed, nthreads):
    """Host-only copy of the tomography workload: operator, phantom, noisy b."""
    from paper_2502_02721_b200.problems import add_noise, random_ellipses  # pure numpy input generators

    key = (grid, angles, bins, seed)
    if key not in _cache:
        _cache.clear()
        t0 = time.perf_counter()
        A, At, m, n = host_tomography(grid, angles, bins, nthreads)
        x = random_ellipses(grid, 10, seed).ravel()
        bc = np.empty(m)
        lib().co_spmv_f32_f64(m, _p(A[0]), _p(A[1]), _p(A[2]), _p(x), _p(bc), nthreads)
        b, _ = add_noise(bc, 0.01, seed + 1)
        _cache[key] = (A, At, m, n, x, b, time.perf_counter() - t0)
    return _cache[key]


_probe = {}


def probe_rate(A, At, m, n, ell, K, nthreads, kpoints=7, S=None):
    """Per-iteration time of the C port over a K-iteration solve: one
    iteration of co_slslu_f32's loop body timed at `kpoints` steps spread over
    k = 1..K (co_probe_iter, with a K-column stand-in basis), interpolated
    piecewise-linearly and averaged over every k.  Returns (rate, ks, times)."""
    L = lib()
    key = (m, n, ell, K)
    if key not in _probe:
        for v in _probe.values():
            L.co_probe_destroy(v[0])
        _probe.clear()
        S = S if S is not None else sparse_sign(ell, m, 8, 7)
        arrs = (np.ascontiguousarray(S.indptr, dtype=np.int64), np.ascontiguousarray(S.indices, dtype=np.int32),
                np.ascontiguousarray(S.data, dtype=np.float64))
        _probe[key] = (L.co_probe_create(m, n, ell, K, nthreads), arrs)
    h, (Srp, Sci, Scv) = _probe[key]
    ks = sorted(set(int(round(v)) for v in np.linspace(1, K, kpoints)))
    times = [L.co_probe_iter(h, k, _p(A[0]), _p(A[1]), _p(A[2]), _p(At[0]), _p(At[1]), _p(At[2]), _p(Srp), _p(Sci),
                             _p(Scv), nthreads) for k in ks]
    mean_t = float(np.mean(np.interp(np.arange(1, K + 1), ks, times)))
    return 1.0 / mean_t, ks, times


def run(w, budget_s=20.0, nthreads=None, b=None, real_iters=4):
    """CPU baseline for a tomography Workload (paper_2502_02721_b200.problems):
    the C port's iteration rate over the config's K iterations (probe_rate),
    plus `real_iters` iterations of the real loop from k = 1 as a check of the
    probe at small k."""
    nthreads = nthreads or os.cpu_count()
    meta = w.meta
    A, At, m, n, x, bh, build_s = host_problem(meta["grid"], meta["angles"], meta["bins"], 0, nthreads)
    K, ell = w.cfg.maxiter, w.cfg.sketch_rows
    S = sparse_sign(ell, m, 8, 7)
    t0 = time.perf_counter()
    rate, ks, times = probe_rate(A, At, m, n, ell, K, nthreads, S=S)
    probe_s = time.perf_counter() - t0
    real = run_slslu(A, At, m, n, bh if b is None else b, ell, real_iters, 1e9, nthreads, S=S) if real_iters else None
    pts = ", ".join(f"k={k}: {t:.3f}s" for k, t in zip(ks, times))
    chk = (f"; real loop k=1..{real['done']}: {np.mean(real['iter_s']):.3f} s/iteration" if real else "")
    return {
        "value": round(rate, 4),
        "unit": "iterations/s",
        "cores": nthreads,
        "kind": "port",
        "nnz": int(A[0][-1]),
        "sample": (f"oracle/coracle.c (C port of solvers.py:410-539, fp32 vectors, OpenMP, QR from scratch and "
                   f"x = L_k y every iteration) on the full {meta['grid']}^2 x {meta['angles']}x{meta['bins']} "
                   f"operator ({int(A[0][-1])} nnz, host-built in {build_s:.1f}s): one iteration timed at each of "
                   f"{len(ks)} steps ({pts}; {probe_s:.1f}s), mean over k=1..{K} by linear interpolation{chk}"),
    }


def psf_conv(img, kernel, nthreads=None):
    """Order-specified zero-boundary convolution (tomo_oracle.psf_stencil,
    transpose=False) of a float32 image, in C."""
    img = np.ascontiguousarray(img, dtype=np.float32)
    K = np.ascontiguousarray(kernel, dtype=np.float32)
    out = np.empty_like(img)
    lib().co_psf_conv_f32(img.shape[0], img.shape[1], _p(K), K.shape[0], K.shape[1], _p(img), _p(out),
                          nthreads or os.cpu_count())
    return out


def scmrh_psf_pivots(shape, kernel, b, maxiter, nthreads=None):
    """The square Hessenberg process (hessenberg.py:160-226) on the PSF
    operator with float32 vectors and basis, in C: (pivots t[:done+1], H)."""
    K = np.ascontiguousarray(kernel, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float64)
    t = np.zeros(maxiter + 1, dtype=np.int64)
    h = np.zeros((maxiter, maxiter + 1))
    done = lib().co_scmrh_psf_f32(shape[0], shape[1], _p(K), K.shape[0], K.shape[1], _p(b), maxiter,
                                  nthreads or os.cpu_count(), _p(t), _p(h))
    return t[: done + 1], np.ascontiguousarray(h[:done].T)
