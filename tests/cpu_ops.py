"""TEST INFRASTRUCTURE: a CPU stand-in for distributed.CudaOps, built from the
oracle, so that the multi-rank orchestration (paper_2512_04317_b200/
distributed.py) can be checked with gloo on CPU.  Each primitive has the
semantics of its CUDA counterpart (include/mxfft_b200.h):
mxfft_fft_rows_scaled, mxfft_prescale_sample_keys, mxfft_prescale_count_range,
mxfft_cabs."""

import numpy as np
import torch

import oracle as O


class SlabPlan:
    """The two plan attributes the orchestration reads, plus the oracle plan."""

    def __init__(self, n, fmt_name="e4m3", block=32):
        self.n = n
        self.stages = n.bit_length() - 1
        self.oplan = O.make_plan(n, O.ALL_MX[fmt_name], block)


def _keys(z: np.ndarray) -> np.ndarray:
    """FP32 squared-magnitude keys as in the kernels: zero -> inf, |re|,|im|
    outside [2^-60, 2^60] -> 0 / 2^125."""
    re = z.real.astype(np.float32).astype(np.float64)
    im = z.imag.astype(np.float32).astype(np.float64)
    k = (re * re + (im * im).astype(np.float32).astype(np.float64)).astype(np.float32)
    m = np.maximum(np.abs(re), np.abs(im))
    k = np.where((m < 2.0**-60) & (m > 0), np.float32(0), k)
    k = np.where(m > 2.0**60, np.float32(2.0**125), k)
    return np.where(m == 0, np.float32(np.inf), k).astype(np.float32)


class OracleOps:
    def rows(self, x, plan, inverse, exp_in=0, exp_out=0):
        a = x.numpy().astype(np.complex128) * 2.0**exp_in
        y = O.fft_batch(a, plan.oplan, inverse).astype(np.complex128) * 2.0**exp_out
        return torch.from_numpy(y.astype(np.complex64))

    def rows_seg(self, recv, plan, inverse, exp_in=0, exp_out=0):
        G, R, _ = recv.shape
        return self.rows(recv.permute(1, 0, 2).reshape(R, G * R).contiguous(), plan, inverse, exp_in, exp_out)

    def sample_keys(self, x, nsamples):
        z = x.numpy()
        nsec = z.size // 4
        j = np.arange(nsamples // 4, dtype=np.uint64)
        h = j * np.uint64(2654435761)
        sec = (h & np.uint64(nsec - 1)) if nsec & (nsec - 1) == 0 else h % np.uint64(nsec)
        idx = (sec[:, None] * np.uint64(4) + np.arange(4, dtype=np.uint64)[None, :]).reshape(-1)
        return torch.from_numpy(_keys(z[idx.astype(np.int64)]))

    def count_range(self, x, lo, hi, top, cand_cap, top_cap):
        z = x.numpy()
        k = _keys(z)
        nz = k != np.inf
        flags = int((~np.isfinite(z)).any() or (k[nz] > 2.0**126).any())
        cm = nz & (k >= np.float32(lo)) & (k <= np.float32(hi))
        tm = nz & (k >= np.float32(top))
        cand, topv = z[cm], z[tm]
        counts = (int(nz.sum()), int((nz & (k < np.float32(lo))).sum()), int(cm.sum()), int(tm.sum()), flags)
        return counts, torch.from_numpy(cand[:cand_cap].copy()), torch.from_numpy(topv[:top_cap].copy())

    def block_transpose(self, a, g):
        R = a.shape[0]
        return torch.from_numpy(np.ascontiguousarray(a.numpy().reshape(R, g, R).transpose(1, 2, 0)))

    def cabs(self, z):
        return torch.from_numpy(O.cabs(z.numpy().astype(np.complex128)))
