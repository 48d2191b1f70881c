"""TEST INFRASTRUCTURE: the statistics kernels' FP32 squared-magnitude keys in
numpy (tests/cpu_ops.py has the same rule): zero -> inf, |re|,|im| outside
[2^-60, 2^60] -> 0 / 2^125."""

import numpy as np


def keys_np(z: np.ndarray) -> np.ndarray:
    re = z.real.astype(np.float32).astype(np.float64)
    im = z.imag.astype(np.float32).astype(np.float64)
    k = (re * re + (im * im).astype(np.float32).astype(np.float64)).astype(np.float32)
    m = np.maximum(np.abs(re), np.abs(im))
    k = np.where((m < 2.0**-60) & (m > 0), np.float32(0), k)
    k = np.where(m > 2.0**60, np.float32(2.0**125), k)
    return np.where(m == 0, np.float32(np.inf), k).astype(np.float32)
