"""Synthetic workloads of BASELINE.json's five configs.

The reference ships only fixed phantoms (problems.py:155-233) and its own
tomography geometry (detectors = grid).  BASELINE's configs ask for seeded
random phantoms and other sizes; the generators here are builder-owned:
every random parameter comes from ``np.random.default_rng(seed)``.  The
operators are the device operators of :mod:`.linops`; ``b = A x_true`` is
applied on the device in float64, and the noise follows the reference's
``add_noise`` (problems.py:353-370).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .linops import DenseOperator, PsfOperator, TomographyOperator
from .solvers import SolverConfig
from .sketch import GaussianSketch, SketchOperator, SparseSignSketch, make_gaussian_sketch

__all__ = [
    "Workload",
    "gaussian_psf",
    "add_noise",
    "toeplitz_blur_1d",
    "bumps_and_step",
    "rectangles_and_discs",
    "random_ellipses",
    "piecewise_constant",
    "make_workload",
    "CONFIGS",
]


def gaussian_psf(sigma, radius=None):
    """problems.py:132-149: normalised separable Gaussian, odd side."""
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


def add_noise(b_clean, level, seed):
    """problems.py:353-370: Gaussian noise rescaled to an exact relative level."""
    b_clean = np.asarray(b_clean, dtype=float)
    if level < 0:
        raise ValueError("noise level must be nonnegative")
    if level == 0:
        return b_clean.copy(), np.zeros_like(b_clean)
    scale = np.linalg.norm(b_clean)
    if scale == 0:
        raise ValueError("relative noise level undefined for a zero vector")
    g = np.random.default_rng(seed).standard_normal(b_clean.size)
    e = (level * scale / np.linalg.norm(g)) * g
    return b_clean + e, e


def toeplitz_blur_1d(n, sigma_frac=0.02):
    """Symmetric Toeplitz Gaussian blur, sigma = sigma_frac * n (index units),
    each row divided by its sum (config 1)."""
    i = np.arange(n, dtype=float)
    s = sigma_frac * n
    A = np.exp(-((i[:, None] - i[None, :]) ** 2) / (2.0 * s * s))
    return A / A.sum(axis=1, keepdims=True)


def bumps_and_step(n, seed):
    """3 Gaussian bumps (random centres, widths, heights) plus one step on [0, 1]."""
    rng = np.random.default_rng(seed)
    t = np.linspace(0.0, 1.0, n)
    x = np.zeros(n)
    for _ in range(3):
        c, w, h = rng.uniform(0.1, 0.9), rng.uniform(0.02, 0.08), rng.uniform(0.5, 1.0)
        x += h * np.exp(-((t - c) ** 2) / (2 * w * w))
    a, hgt = rng.uniform(0.2, 0.8), rng.uniform(0.3, 0.7)
    x += hgt * (t >= a)
    return x


def rectangles_and_discs(size, count, seed):
    """``count`` random axis-aligned rectangles and discs, intensities U(0,1), additive."""
    rng = np.random.default_rng(seed)
    r, c = np.mgrid[0:size, 0:size].astype(float) / size
    img = np.zeros((size, size))
    for i in range(count):
        v = rng.uniform(0.0, 1.0)
        if i % 2 == 0:
            r0, c0 = rng.uniform(0, 0.8, size=2)
            h, w = rng.uniform(0.05, 0.3, size=2)
            img[(r >= r0) & (r < r0 + h) & (c >= c0) & (c < c0 + w)] += v
        else:
            cr, cc = rng.uniform(0.1, 0.9, size=2)
            rad = rng.uniform(0.03, 0.15)
            img[(r - cr) ** 2 + (c - cc) ** 2 <= rad * rad] += v
    return img


def random_ellipses(grid, count, seed):
    """``count`` random ellipses with additive densities U(0,1) inside the unit disc."""
    rng = np.random.default_rng(seed)
    y, x = (np.mgrid[0:grid, 0:grid].astype(np.float64) + 0.5) / grid * 2.0 - 1.0
    img = np.zeros((grid, grid))
    for _ in range(count):
        cx, cy = rng.uniform(-0.5, 0.5, size=2)
        a, b = rng.uniform(0.1, 0.45, size=2)
        th = rng.uniform(0, math.pi)
        v = rng.uniform(0.0, 1.0)
        ct, st = math.cos(th), math.sin(th)
        xr = (x - cx) * ct + (y - cy) * st
        yr = -(x - cx) * st + (y - cy) * ct
        img[(xr / a) ** 2 + (yr / b) ** 2 <= 1.0] += v
    return img


def piecewise_constant(size, seed, blocks=16):
    """Seeded piecewise-constant image: a random ``blocks`` x ``blocks`` grid of
    levels U(0,1) with a few random discs on top."""
    rng = np.random.default_rng(seed)
    levels = rng.uniform(0.0, 1.0, size=(blocks, blocks))
    img = np.kron(levels, np.ones((size // blocks + 1, size // blocks + 1)))[:size, :size].copy()
    r, c = np.mgrid[0:size, 0:size].astype(np.float32) / size
    for _ in range(8):
        cr, cc = rng.uniform(0.1, 0.9, size=2)
        rad = rng.uniform(0.03, 0.12)
        img[(r - cr) ** 2 + (c - cc) ** 2 <= rad * rad] = rng.uniform(0.0, 1.0)
    return img


@dataclass
class Workload:
    name: str
    solver: str          # "scmrh" or "slslu"
    operator: object
    b: np.ndarray
    x_true: np.ndarray
    cfg: SolverConfig
    sketch: object = None   # SketchOperator for S2
    meta: dict = field(default_factory=dict)


CONFIGS = {
    1: "1D deblurring, dense fp64 1024^2 Toeplitz (sigma=0.02 n), sCMRH K=100, Gaussian s=400",
    2: "2D deblurring 256^2, 15x15 PSF (sigma=2), fp32, sCMRH K=200, Gaussian s=800",
    3: "tomography 512^2, 180 angles x 725 bins, CSR fp32, sLSLU lam=1e-3 K=200, sparse-sign s=800 zeta=8",
    4: "tomography 2048^2, 720 angles x 2897 bins, CSR fp32, sLSLU K=300, sparse-sign s=1200 zeta=8",
    5: "deblurring 4096^2, 31x31 PSF (sigma=4), bf16 basis / fp32 work, sCMRH K=150, Gaussian s=600",
}


def make_workload(cfg_id, seed=0, scale=None, maxiter=None):
    """Build config ``cfg_id`` (1-5).  ``scale`` shrinks the image side of
    configs 2-5 (tests); ``maxiter`` overrides K (the sketch size keeps the
    config's rule, at least maxiter+1)."""
    if cfg_id == 1:
        n = 1024 if scale is None else int(scale)
        A = toeplitz_blur_1d(n)
        op = DenseOperator(A)
        x = bumps_and_step(n, seed)
        b, _ = add_noise(A @ x, 0.01, seed + 1)
        K = maxiter or 100
        cfg = SolverConfig(maxiter=K, sketch_rows=max(4 * 100, K + 1), seed=seed, sketch_kind="pcg64")
        return Workload("cfg1", "scmrh", op, b, x, cfg)
    if cfg_id == 2:
        size = 256 if scale is None else int(scale)
        psf = gaussian_psf(2.0, radius=7)
        op = PsfOperator(size, psf, dtype=np.float32)
        x = rectangles_and_discs(size, 20, seed).ravel()
        b, _ = add_noise(op.matvec(x), 0.01, seed + 1)
        K = maxiter or 200
        cfg = SolverConfig(maxiter=K, sketch_rows=max(800, K + 1), seed=seed, dtype="float32", sketch_kind="gaussian")
        return Workload("cfg2", "scmrh", op, b, x, cfg, meta={"image": (size, size)})
    if cfg_id in (3, 4):
        if cfg_id == 3:
            grid, angles, bins, K, ell, lam = 512, 180, 725, 200, 800, 1e-3
        else:
            grid, angles, bins, K, ell, lam = 2048, 720, 2897, 300, 1200, 0.0
        if scale is not None:
            f = int(scale) / grid
            grid = int(scale)
            angles = max(2, int(round(angles * f)))
            bins = max(2, int(round(bins * f)))
        K = maxiter or K
        op = TomographyOperator(grid, angles, bins, dtype=np.float32)
        x = random_ellipses(grid, 10, seed).ravel()
        b, _ = add_noise(op.matvec(x), 0.01, seed + 1)
        ell = max(ell, K + 1)
        S2 = SparseSignSketch(ell, op.rows, seed=seed + 7, zeta=8)
        cfg = SolverConfig(maxiter=K, sketch_rows=ell, seed=seed, lam=lam, dtype="float32", sketch_kind="gaussian")
        return Workload(f"cfg{cfg_id}", "slslu", op, b, x, cfg,
                        sketch=SketchOperator(ell, op.rows, seed + 7, S2),
                        meta={"grid": grid, "angles": angles, "bins": bins, "nnz": op.info()["nnz"]})
    if cfg_id == 5:
        size = 4096 if scale is None else int(scale)
        psf = gaussian_psf(4.0, radius=15)
        op = PsfOperator(size, psf, dtype=np.float32)
        x = piecewise_constant(size, seed).ravel()
        b, _ = add_noise(op.matvec(x), 0.005, seed + 1)
        K = maxiter or 150
        cfg = SolverConfig(maxiter=K, sketch_rows=max(600, K + 1), seed=seed, dtype="float32",
                           basis_dtype="bfloat16", sketch_kind="gaussian")
        return Workload("cfg5", "scmrh", op, b, x, cfg, meta={"image": (size, size)})
    raise ValueError(f"unknown config {cfg_id}")
