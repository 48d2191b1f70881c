"""Seeded synthetic k-space inputs (host-side generator for tests and bench).

The reference measures on MRI datasets (fastMRI, SKM-TEA) that are not in this
container; BASELINE.json fixes a seeded ellipse phantom instead:

* phantom: real N x N image, K ~ U{8..16} filled ellipses; intensity
  U[0.1, 1]; centres U(-0.7, 0.7)^2 and semi-axes U(0.05, 0.5) in a [-1, 1)^2
  field of view; rotation U[0, pi); overlaps add;
* k-space = fftshift(fft2(phantom)) in FP64, plus complex Gaussian noise with
  per-component sigma = noise * max|k| / sqrt(2) (noise = 0.01 default, 0.05 for
  the 4096 x 128^2 config), so the complex noise RMS is noise * peak;
* cast to complex64 once: the GPU and the CPU oracle see identical values.

This is input generation only (not the transform under test); it uses numpy's
own FFT to build the k-space.
"""

from __future__ import annotations

import numpy as np


def ellipse_phantom(n: int, rng: np.random.Generator) -> np.ndarray:
    ax = (np.arange(n) - n / 2) / (n / 2)
    yy, xx = np.meshgrid(ax, ax, indexing="ij")
    img = np.zeros((n, n))
    for _ in range(int(rng.integers(8, 17))):
        amp = rng.uniform(0.1, 1.0)
        cx, cy = rng.uniform(-0.7, 0.7, size=2)
        a, b = rng.uniform(0.05, 0.5, size=2)
        th = rng.uniform(0.0, np.pi)
        c, s = np.cos(th), np.sin(th)
        u = (xx - cx) * c + (yy - cy) * s
        v = -(xx - cx) * s + (yy - cy) * c
        img[(u / a) ** 2 + (v / b) ** 2 <= 1.0] += amp
    return img


def ellipse_kspace(n: int, seed: int, noise: float = 0.01) -> np.ndarray:
    """One seeded complex64 k-space image (n, n)."""
    rng = np.random.default_rng(seed)
    k = np.fft.fftshift(np.fft.fft2(ellipse_phantom(n, rng)))
    sigma = noise * float(np.abs(k).max()) / np.sqrt(2.0)
    k = k + sigma * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    return k.astype(np.complex64)


def ellipse_kspace_batch(batch: int, n: int, seed: int = 0, noise: float = 0.01) -> np.ndarray:
    """(batch, n, n) complex64; image i uses seed + i."""
    out = np.empty((batch, n, n), dtype=np.complex64)
    for i in range(batch):
        out[i] = ellipse_kspace(n, seed + i, noise)
    return out


def ellipse_kspace_device(n: int, seed: int, noise: float = 0.01, device="cuda", rows=None):
    """The same kind of seeded phantom k-space, synthesised on the GPU with
    torch (for C5's 16384^2 image, where the host generator needs minutes and
    4 GiB).  Ellipse parameters come from the same numpy stream as
    ellipse_phantom; the FFT is torch.fft in FP64, noise from a seeded torch
    generator.  Not bit-identical to ellipse_kspace (input synthesis only).
    rows = (r0, r1) returns just those rows of the image (a row slab)."""
    import torch

    rng = np.random.default_rng(seed)
    params = []
    for _ in range(int(rng.integers(8, 17))):
        amp = rng.uniform(0.1, 1.0)
        cx, cy = rng.uniform(-0.7, 0.7, size=2)
        a, b = rng.uniform(0.05, 0.5, size=2)
        th = rng.uniform(0.0, np.pi)
        params.append((amp, cx, cy, a, b, np.cos(th), np.sin(th)))
    ax = (torch.arange(n, device=device, dtype=torch.float64) - n / 2) / (n / 2)
    img = torch.zeros((n, n), dtype=torch.float64, device=device)
    step = max(1, (1 << 24) // n)
    for r0 in range(0, n, step):  # rasterise in row blocks to bound temporaries
        yy = ax[r0:r0 + step, None]
        xx = ax[None, :]
        blk = img[r0:r0 + step]
        for amp, cx, cy, a, b, c, s in params:
            u = (xx - cx) * c + (yy - cy) * s
            v = -(xx - cx) * s + (yy - cy) * c
            blk += amp * ((u / a) ** 2 + (v / b) ** 2 <= 1.0)
    k = torch.fft.fftshift(torch.fft.fft2(img))
    del img
    sigma = noise * float(k.abs().max()) / np.sqrt(2.0)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    r0, r1 = rows if rows is not None else (0, n)
    ks = k[r0:r1]
    out = (ks + sigma * torch.complex(torch.randn(ks.shape, generator=g, device=device, dtype=torch.float64),
                                      torch.randn(ks.shape, generator=g, device=device,
                                                  dtype=torch.float64))).to(torch.complex64)
    return out.contiguous()
