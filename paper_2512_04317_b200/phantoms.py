"""TRANSCRIPTION, labelled as such: gen_phantom / coil_sensitivities /
_phantom_magnitude follow the reference's host generators
(pkg/src/mxfft/mri.py:115-195) statement by statement -- same constants, same
RNG draw order -- because their outputs must be identical grids.  This is
host-only input synthesis, kept only so that the
reference's public names resolve (drop-in completeness); it is not part of the
B200 hot path and claims no credit.  The one piece that runs on the GPU is the
k-space step, the FP64 reference-mode transform (csrc/mxfft_modes.cu)."""

from __future__ import annotations

import math

import numpy as np

from .errors import ConfigError
from .fftcore import ModeSpec, fft_2d, make_plan


def _grid(n: int):
    """(yy, xx) on [-1, 1]^2, 'ij' indexing."""
    ax = np.linspace(-1.0, 1.0, n)
    return np.meshgrid(ax, ax, indexing="ij")


def coil_sensitivities(n: int, coils: int, seed: int) -> np.ndarray:
    """(coils, n, n) smooth complex coil maps; |map| >= 0.6 everywhere."""
    rng = np.random.default_rng(seed + 7919)
    yy, xx = _grid(n)
    maps = np.empty((coils, n, n), dtype=np.complex128)
    for c in range(coils):
        theta = 2.0 * np.pi * c / coils
        cx, cy = 0.6 * math.cos(theta), 0.6 * math.sin(theta)
        bump = np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * 0.5**2))
        gx, gy = rng.uniform(-1.5, 1.5, size=2)
        maps[c] = (0.6 + 0.9 * bump) * np.exp(1j * (gx * xx + gy * yy))
    return maps


def _magnitude(n: int, kind: str, rng, tail: float) -> np.ndarray:
    yy, xx = _grid(n)
    edge = 0.5 * (1.0 + np.tanh((0.85 - np.sqrt(xx**2 + yy**2)) / 0.05))
    if kind == "blobs":
        mag = np.zeros((n, n))
        for _ in range(6):
            cx, cy = rng.uniform(-0.5, 0.5, size=2)
            width = rng.uniform(0.08, 0.25)
            height = rng.uniform(0.4, 1.0)
            mag += height * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * width**2))
    elif kind == "bars":
        theta = rng.uniform(0, np.pi)
        period = rng.uniform(0.15, 0.35)
        offset = rng.uniform(0, 2 * np.pi)
        ramp = (xx * math.cos(theta) + yy * math.sin(theta)) / period
        mag = 0.55 + 0.45 * np.tanh(4.0 * np.sin(2 * np.pi * ramp + offset))
    else:
        raise ConfigError("kind", f"unknown phantom kind {kind!r}")
    if tail > 0:
        from scipy.ndimage import gaussian_filter

        mag = mag + tail * np.abs(gaussian_filter(rng.standard_normal((n, n)), sigma=1.0))
    return mag * edge


def gen_phantom(n: int, coils: int, seed: int, kind: str = "blobs", tail: float = 0.0, noise: float = 1e-4):
    """(image grid, k-space grid) of a seeded multi-coil phantom; the k-space is
    the exact FP64 inverse transform / N^2 of the coil images."""
    from .mri import IMAGE, KSPACE, ComplexGrid

    if n < 2 or n & (n - 1):
        raise ConfigError("n", "must be a power of two >= 2")
    if coils < 1:
        raise ConfigError("coils", "must be >= 1")
    rng = np.random.default_rng(seed)
    mag = _magnitude(n, kind, rng, tail)
    yy, xx = _grid(n)
    a, b, c, d = rng.uniform(-1.0, 1.0, size=4)
    phase = np.pi * (a * xx + b * yy + c * xx * yy + d * (xx**2 - yy**2))
    img = mag * np.exp(1j * phase) * coil_sensitivities(n, coils, seed)
    if noise > 0:
        img = img + noise * (rng.standard_normal((coils, n, n)) + 1j * rng.standard_normal((coils, n, n)))
    plan = make_plan(n, ModeSpec.reference())
    scale = 1.0 / (n * n)
    ksp = np.stack([fft_2d(img[i], plan, "inverse") * scale for i in range(coils)])
    return ComplexGrid(img, IMAGE), ComplexGrid(ksp, KSPACE)
