"""TEST INFRASTRUCTURE ONLY -- numpy restatements of the operators the device
kernels must reproduce.

* ``trace_ray`` / ``tomography_matrix``: the reference's exact-chord
  parallel-beam projector (problems.py:276-331), generalised from
  ``detector_count == grid`` to an arbitrary detector count ``n_bins`` with
  offsets ``s_j = j + 0.5 - n_bins / 2`` (with ``n_bins == grid`` this is the
  reference formula, problems.py:319-331, and the fixtures pin it bitwise).
* ``psf_stencil``: a tap-ordered 2-D zero-boundary convolution / correlation.
  The reference calls scipy ``convolve2d``/``correlate2d`` (problems.py:257-267)
  whose summation order is internal to scipy; this stencil fixes the order
  (rows of taps a = 0..kh-1 outer, b = 0..kw-1 inner, starting from +0, product
  rounded then added, zero padding contributes ``K * 0``) and is checked against
  scipy to <= 1e-14 relative in the tests.
* ``gaussian_psf``: problems.py:132-149.
* ``add_noise``: problems.py:353-370.

Not a product path.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.sparse


def trace_ray(origin, direction, grid):
    """problems.py:276-308: exact intersection lengths of one ray with the
    grid's pixels; returns (flat pixel indices in traversal order, lengths)."""
    t0, t1 = -np.inf, np.inf
    for axis in range(2):
        o, d = origin[axis], direction[axis]
        if abs(d) < 1e-12:
            if o <= 0.0 or o >= grid:
                return np.empty(0, dtype=np.int64), np.empty(0)
        else:
            ta, tb = (0.0 - o) / d, (grid - o) / d
            if ta > tb:
                ta, tb = tb, ta
            t0, t1 = max(t0, ta), min(t1, tb)
    if not t1 > t0:
        return np.empty(0, dtype=np.int64), np.empty(0)
    crossings = [np.array([t0, t1])]
    for axis in range(2):
        o, d = origin[axis], direction[axis]
        if abs(d) >= 1e-12:
            t = (np.arange(1.0, grid) - o) / d
            crossings.append(t[(t > t0) & (t < t1)])
    alphas = np.unique(np.concatenate(crossings))
    lengths = np.diff(alphas)
    mids = origin[None, :] + (0.5 * (alphas[:-1] + alphas[1:]))[:, None] * direction
    ci = np.clip(np.floor(mids[:, 0]).astype(np.int64), 0, grid - 1)
    rj = np.clip(np.floor(mids[:, 1]).astype(np.int64), 0, grid - 1)
    keep = lengths > 1e-12
    return rj[keep] * grid + ci[keep], lengths[keep]


def ray_geometry(grid, n_angles, n_bins=None):
    """Angle table and detector offsets exactly as problems.py:317-322 forms
    them (``math.pi * a / n_angles``, ``math.cos``/``math.sin``)."""
    n_bins = grid if n_bins is None else int(n_bins)
    cos_t = np.empty(n_angles)
    sin_t = np.empty(n_angles)
    for a in range(n_angles):
        theta = math.pi * a / n_angles
        cos_t[a] = math.cos(theta)
        sin_t[a] = math.sin(theta)
    offsets = np.array([j + 0.5 - n_bins / 2.0 for j in range(n_bins)])
    return cos_t, sin_t, offsets


def tomography_matrix(grid, n_angles, n_bins=None, rows=None):
    """problems.py:311-331 with a detector count ``n_bins`` (default ``grid``).

    Row ``a * n_bins + j`` holds the chord lengths of detector j at angle a.
    ``rows`` optionally restricts the assembly to a subset of ray indices
    (the matrix keeps its full shape; other rows are empty).
    Returns a canonical float64 CSR (sorted indices, duplicates summed)."""
    n_bins = grid if n_bins is None else int(n_bins)
    centre = np.array([grid / 2.0, grid / 2.0])
    cos_t, sin_t, offsets = ray_geometry(grid, n_angles, n_bins)
    want = None if rows is None else set(int(r) for r in rows)
    rr, cc, vv = [], [], []
    for a in range(n_angles):
        direction = np.array([cos_t[a], sin_t[a]])
        normal = np.array([-sin_t[a], cos_t[a]])
        for j in range(n_bins):
            r = a * n_bins + j
            if want is not None and r not in want:
                continue
            origin = centre + offsets[j] * normal
            idx, lengths = trace_ray(origin, direction, grid)
            rr.extend([r] * idx.size)
            cc.extend(idx.tolist())
            vv.extend(lengths.tolist())
    M = scipy.sparse.csr_matrix(
        (np.asarray(vv, dtype=np.float64), (np.asarray(rr, dtype=np.int64), np.asarray(cc, dtype=np.int64))),
        shape=(n_angles * n_bins, grid * grid),
    )
    M.sum_duplicates()
    M.sort_indices()
    return M


def csr_sequential_matvec(indptr, indices, data, x, dtype):
    """The scipy csr_matvec order: per row, acc = 0; acc = acc + v * x[col]
    left to right, product rounded then added (no FMA)."""
    dtype = np.dtype(dtype)
    y = np.zeros(len(indptr) - 1, dtype=dtype)
    x = np.asarray(x, dtype=dtype)
    data = np.asarray(data, dtype=dtype)
    for i in range(len(indptr) - 1):
        acc = dtype.type(0.0)
        for p in range(indptr[i], indptr[i + 1]):
            acc = dtype.type(acc + dtype.type(data[p] * x[indices[p]]))
        y[i] = acc
    return y


def gaussian_psf(sigma, radius=None):
    """problems.py:132-149."""
    if sigma < 0:
        raise ValueError("sigma must be nonnegative")
    if sigma == 0:
        return np.ones((1, 1))
    if radius is None:
        radius = max(1, math.ceil(3.0 * sigma))
    d = np.arange(-radius, radius + 1, dtype=float)
    g = np.exp(-(d**2) / (2.0 * sigma**2))
    kernel = np.outer(g, g)
    return kernel / kernel.sum()


def psf_stencil(img, kernel, transpose=False, dtype=np.float64):
    """Tap-ordered zero-boundary 'same' convolution (transpose=False) or
    correlation (transpose=True) of a (H, W) image.

    out[r, c] = sum over a (outer), b (inner) of K[a, b] * xpad[...] with
      convolution:  x[r + ry - a, c + rx - b]
      correlation:  x[r - ry + a, c - rx + b]
    where (ry, rx) = kernel half sizes; each product is rounded then added to
    the running sum (no FMA), starting from +0.  Vectorised over pixels, so
    the per-pixel operation sequence is exactly the device kernel's."""
    dtype = np.dtype(dtype)
    img = np.asarray(img, dtype=dtype)
    K = np.asarray(kernel, dtype=dtype)
    kh, kw = K.shape
    ry, rx = kh // 2, kw // 2
    H, W = img.shape
    pad = np.zeros((H + 2 * ry, W + 2 * rx), dtype=dtype)
    pad[ry:ry + H, rx:rx + W] = img
    out = np.zeros((H, W), dtype=dtype)
    for a in range(kh):
        for b in range(kw):
            if transpose:
                sl = pad[a:a + H, b:b + W]
            else:
                sl = pad[2 * ry - a:2 * ry - a + H, 2 * rx - b:2 * rx - b + W]
            out = out + K[a, b] * sl
    return out


def add_noise(b_clean, level, seed):
    """problems.py:353-370: Gaussian noise rescaled to an exact relative level."""
    b_clean = np.asarray(b_clean, dtype=float)
    if level < 0:
        raise ValueError("noise level must be nonnegative")
    if level == 0:
        return b_clean.copy(), np.zeros_like(b_clean)
    scale = np.linalg.norm(b_clean)
    g = np.random.default_rng(seed).standard_normal(b_clean.size)
    e = (level * scale / np.linalg.norm(g)) * g
    return b_clean + e, e
