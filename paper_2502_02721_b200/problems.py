"""Problem builders: the reference's own (``make_tomography``, ``make_deblur``,
their phantoms and PSFs, the ``Problem`` / ``Image`` bundles and 16-bit PGM
image exchange, problems.py:61-473) with device operators, and the synthetic
workloads of BASELINE.json's five configs.

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

from typing import Optional

from .linops import DenseOperator, PsfOperator, TomographyOperator
from .solvers import SolverConfig
from .sketch import GaussianSketch, SketchOperator, SparseSignSketch, make_gaussian_sketch

__all__ = [
    "Problem",
    "Image",
    "ImageFormatError",
    "motion_psf",
    "deblur_phantom",
    "tomography_phantom",
    "make_deblur",
    "make_tomography",
    "image_from_vector",
    "write_image",
    "read_image",
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


# ---------------------------------------------------------------------------
# the reference's problem bundles, phantoms and builders (problems.py:61-351)


@dataclass
class Problem:
    """``b = A x_true + e`` (problems.py:61-99); ``operator`` is a device operator."""

    operator: object
    b: np.ndarray
    x_true: Optional[np.ndarray] = None
    noise_level: float = 0.0
    seed: int = 0
    image_shape: Optional[tuple] = None

    def __post_init__(self):
        self.b = np.asarray(self.b, dtype=float)
        if self.b.ndim != 1 or self.b.size != self.operator.rows:
            raise ValueError("observation length must match operator rows")
        if self.x_true is not None:
            self.x_true = np.asarray(self.x_true, dtype=float)
            if self.x_true.ndim != 1 or self.x_true.size != self.operator.cols:
                raise ValueError("ground truth length must match operator cols")
        if self.noise_level < 0:
            raise ValueError("noise level must be nonnegative")


@dataclass
class Image:
    """Grayscale image in [0, 1], row-major ``pixels[height, width]``, row 0
    at the top (problems.py:101-121)."""

    width: int
    height: int
    pixels: np.ndarray

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be positive")
        self.pixels = np.asarray(self.pixels, dtype=float)
        if self.pixels.shape != (self.height, self.width):
            raise ValueError("pixel array must have shape (height, width)")
        if not np.all(np.isfinite(self.pixels)):
            raise ValueError("pixel values must be finite")
        if self.pixels.min() < 0.0 or self.pixels.max() > 1.0:
            raise ValueError("pixel values must lie in [0, 1]")


class ImageFormatError(ValueError):
    """Malformed image file; the message names a byte offset (problems.py:124-125)."""


def motion_psf(length, angle_deg, oversample=64):
    """Unit-mass motion-blur segment (problems.py:152-189): ``round(length *
    oversample) + 1`` (at least 2) points along a centred segment at
    ``angle_deg`` from the horizontal, each deposited bilinearly on the odd
    ``2 ceil((length-1)/2) + 1`` square; axis directions snapped."""
    if length < 1:
        raise ValueError("length must be at least 1")
    if not np.isfinite(angle_deg):
        raise ValueError("angle must be finite")
    half = math.ceil((length - 1.0) / 2.0)
    side = 2 * half + 1
    out = np.zeros((side, side))
    th = math.radians(angle_deg)
    ux, uy = math.cos(th), math.sin(th)
    if abs(ux) < 1e-12:
        ux = 0.0
    if abs(uy) < 1e-12:
        uy = 0.0
    npts = max(2, int(round(length * oversample)) + 1)
    span = (length - 1.0) / 2.0
    for t in np.linspace(-span, span, npts):
        py, px = half + t * uy, half + t * ux
        iy, ix = int(math.floor(py)), int(math.floor(px))
        fy, fx = py - iy, px - ix
        taps = ((iy, ix, (1 - fy) * (1 - fx)), (iy, ix + 1, (1 - fy) * fx),
                (iy + 1, ix, fy * (1 - fx)), (iy + 1, ix + 1, fy * fx))
        for r, c, wgt in taps:
            if wgt > 0 and 0 <= r < side and 0 <= c < side:
                out[r, c] += wgt
    return out / out.sum()


def deblur_phantom(size):
    """Fixed deblurring test image (problems.py:192-209): gradient background
    0.10..0.35, rectangle 0.85, discs 0.70 / 0.05, vertical bar 0.95."""
    s = size
    rr, cc = np.mgrid[0:s, 0:s].astype(float)
    img = 0.10 + 0.25 * cc / max(s - 1, 1)
    img[int(0.15 * s): int(0.45 * s), int(0.20 * s): int(0.55 * s)] = 0.85
    for (cy, cx, rad, val) in ((0.62, 0.40, 0.18, 0.70), (0.30, 0.70, 0.08, 0.05)):
        img[(rr - cy * s) ** 2 + (cc - cx * s) ** 2 <= (rad * s) ** 2] = val
    w = max(1, s // 32)
    img[int(0.55 * s): int(0.90 * s), int(0.78 * s): int(0.78 * s) + w] = 0.95
    return img


def tomography_phantom(grid):
    """Fixed absorption phantom (problems.py:212-233): discs 0.55, 1.0, 0.30
    and a 0.0 void, painted in order on a zero background (pixel centres)."""
    g = grid
    rr, cc = np.mgrid[0:g, 0:g] + 0.5
    img = np.zeros((g, g))
    for cy, cx, rad, val in ((0.50, 0.50, 0.38, 0.55), (0.40, 0.42, 0.13, 1.00),
                             (0.63, 0.58, 0.10, 0.30), (0.52, 0.33, 0.05, 0.00)):
        img[(rr - cy * g) ** 2 + (cc - cx * g) ** 2 <= (rad * g) ** 2] = val
    return img


def make_deblur(size, psf, noise_level=0.0, seed=0):
    """problems.py:240-273 on the device: zero-boundary convolution operator
    (:class:`PsfOperator`, fp64; transpose = correlation), the fixed phantom,
    b = A x_true + exact-level noise.  The stencil sums taps in a fixed order,
    so b agrees with scipy's ``convolve2d`` to ~1e-16 relative, not bitwise
    (SURVEY.md 8a item 7)."""
    if size < 8:
        raise ValueError("size must be at least 8")
    k = np.asarray(psf, dtype=float)
    if k.ndim != 2 or k.shape[0] % 2 == 0 or k.shape[1] % 2 == 0:
        raise ValueError("psf must be a 2-D kernel with odd side lengths")
    if k.shape[0] >= size or k.shape[1] >= size:
        raise ValueError("psf support must be smaller than the image")
    op = PsfOperator((size, size), k, dtype=np.float64)
    x_true = deblur_phantom(size).ravel()
    b, _ = add_noise(op.matvec(x_true), noise_level, seed)
    return Problem(op, b, x_true, noise_level, seed, (size, size))


def make_tomography(grid, n_angles, noise_level=0.0, seed=0):
    """problems.py:334-350 on the device: the exact-chord parallel-beam matrix
    (``grid`` detectors, built by the device ray tracer bit-identically to
    ``tomography_matrix``), the fixed phantom, b = K x_true (bitwise the
    reference's scipy product) + exact-level noise."""
    if grid < 8:
        raise ValueError("grid must be at least 8")
    if n_angles < 2:
        raise ValueError("need at least 2 angles")
    op = TomographyOperator(grid, n_angles, dtype=np.float64)
    x_true = tomography_phantom(grid).ravel()
    b, _ = add_noise(op.matvec(x_true), noise_level, seed)
    return Problem(op, b, x_true, noise_level, seed, (grid, grid))


# ---------------------------------------------------------------------------
# 16-bit binary PGM exchange (problems.py:377-473)


def image_from_vector(v, height, width, clip=True):
    """Flat solution vector -> :class:`Image` (clipped to [0, 1] by default)."""
    px = np.asarray(v, dtype=float).reshape(height, width)
    return Image(width=width, height=height, pixels=np.clip(px, 0.0, 1.0) if clip else px)


def write_image(image, path):
    """P5 PGM, maxval 65535, big-endian samples round(clip(p) * 65535)."""
    q = np.round(np.clip(image.pixels, 0.0, 1.0) * 65535.0).astype(">u2")
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n65535\n" % (image.width, image.height))
        fh.write(q.tobytes())


def _pgm_header(data):
    """Parse the P5 header; returns (width, height, maxval, sample offset).
    Whitespace and '#' comments separate tokens; errors name the byte offset."""
    pos = 0

    def err(what, at):
        raise ImageFormatError(f"{what} at byte offset {at}")

    def skip(p):
        while p < len(data):
            ch = data[p:p + 1]
            if ch.isspace():
                p += 1
            elif ch == b"#":
                while p < len(data) and data[p:p + 1] not in (b"\n", b"\r"):
                    p += 1
            else:
                break
        return p

    def token(p):
        p = skip(p)
        q = p
        while q < len(data) and not data[q:q + 1].isspace():
            q += 1
        if q == p:
            err("unexpected end of header", p)
        return data[p:q], p, q

    tok, start, pos = token(pos)
    if tok != b"P5":
        err("missing P5 magic token", 0)
    vals = []
    for what in ("width", "height", "maximum sample value"):
        tok, start, pos = token(pos)
        try:
            v = int(tok)
        except ValueError:
            err(f"invalid {what} {tok!r}", start)
        if v < 1:
            err(f"nonpositive {what}", start)
        vals.append(v)
    width, height, maxval = vals
    if maxval > 65535:
        err("maximum sample value above 65535", pos)
    if pos >= len(data) or not data[pos:pos + 1].isspace():
        err("missing separator before samples", pos)
    return width, height, maxval, pos + 1


def read_image(path):
    """Binary PGM (P5, 8- or 16-bit samples, maxval <= 65535) -> :class:`Image`
    scaled to [0, 1]; malformed files raise :class:`ImageFormatError`."""
    with open(path, "rb") as fh:
        data = fh.read()
    width, height, maxval, off = _pgm_header(data)
    dt = np.dtype(">u2" if maxval > 255 else "u1")
    need = width * height * dt.itemsize
    if len(data) - off < need:
        raise ImageFormatError(f"truncated sample data at byte offset {len(data)}")
    samples = np.frombuffer(data[off:off + need], dtype=dt).astype(float)
    return Image(width=width, height=height, pixels=(samples / maxval).reshape(height, width))


# ---------------------------------------------------------------------------
# BASELINE workloads


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
