"""TEST INFRASTRUCTURE: a CPU stand-in for distributed.CudaOps, built from the
oracle, so that the multi-rank orchestration (paper_2512_04317_b200/
distributed.py) can be checked with gloo on CPU.  Each primitive has the
semantics of its CUDA counterpart (include/mxfft_b200.h):
mxfft_fft_rows_scaled, mxfft_prescale_sample_keys, mxfft_prescale_count_range,
mxfft_cabs, and the folded prescale's mxfft_fft_rows_evidence /
mxfft_fold_reduce / mxfft_fold_finish (same words, same decision rule; the
block-exponent range, which only the kernel sees, is reported as [0, 0])."""

import math

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


    # ---- the folded prescale (distributed.prescale_fold_slab) ----
    def rows_evidence(self, x, plan, inverse=False):
        y = self.rows(x, plan, inverse)
        z = x.numpy().reshape(-1)
        re = z.real.astype(np.float32)
        im = z.imag.astype(np.float32)
        t = (im.astype(np.float64) * im.astype(np.float64)).astype(np.float32)
        key = (re.astype(np.float64) * re.astype(np.float64) + t.astype(np.float64)).astype(np.float32)
        mu = np.maximum(np.abs(re), np.abs(im)).view(np.uint32).astype(np.int64)
        g32 = mu.reshape(-1, 32)  # any partition of the points into 32s serves as the "threads"
        zeros = (g32 == 0).sum(1)
        mn = np.where(g32 == 0, 1 << 40, g32).min(1)
        thread_words = np.where(mn >= (1 << 40), 0xFFFFFFC0, mn & ~63) | zeros
        kmax = key.view(np.uint32).reshape(-1, 1024).max(1).astype(np.int64)
        warp_words = np.stack([kmax, np.full_like(kmax, (128 << 16) | (128 << 4))], 1).reshape(-1)
        words = np.concatenate([warp_words, thread_words]).astype(np.uint32)
        return y, torch.from_numpy(words.view(np.uint8).copy())

    @staticmethod
    def _k1(kmx, cfg):
        a_est = math.sqrt(float(np.array(kmx, dtype=np.uint32).view(np.float32)))
        L1 = math.log2(cfg.target / max(a_est, 1e-30)) if a_est > 0 else float("inf")
        e_key = (kmx >> 23) - 127
        ok = kmx < 0x7F800000 and e_key >= -100 and math.isfinite(L1) and abs(abs(L1 - math.trunc(L1)) - 0.5) > 1e-6
        k1 = (math.floor(L1 + 0.5) if L1 >= 0 else math.ceil(L1 - 0.5)) if ok else 0
        T = np.float32(np.nextafter(np.float32(math.ldexp(cfg.tau_min, -k1) * (1 + 2.0**-20)), np.float32(np.inf))) if ok else np.float32(0)
        return a_est, k1, e_key, ok, T

    def fold_reduce(self, words, npoints, cfg, step, g=None):
        w = words.numpy().view(np.uint32).astype(np.int64)
        nw = npoints // 512
        if step == 0:
            ww = w[:nw].reshape(-1, 2)
            vals = [ww[:, 0].max(), (ww[:, 1] >> 16).max(), ((ww[:, 1] >> 4) & 0xFFF).max(), (ww[:, 1] & 1).max(), 0, 0, 0, 0]
            return torch.from_numpy(np.array(vals, dtype=np.int64).astype(np.uint32).view(np.int32).copy())
        gv = g.numpy().view(np.uint32)
        _, _, _, _, T = self._k1(int(gv[0]), cfg)
        tw = w[nw:nw + npoints // 32]
        mb = tw & ~63
        live = mb != 0xFFFFFFC0
        small = int((live & (mb.astype(np.uint32).view(np.float32) < T)).sum())
        mn = int(mb[live].min()) if live.any() else 0xFFFFFFFF
        gv[4], gv[5], gv[6] = int((tw & 63).sum()), small, (~mn) & 0xFFFFFFFF
        return g

    def fold_finish(self, g, total_points, cfg):
        from paper_2512_04317_b200 import _native

        gv = [int(v) for v in g.numpy().view(np.uint32)]
        kmx, hi, lo, rep, zeros, small, mn = gv[0], gv[1] - 128, 128 - gv[2], gv[3], gv[4], gv[5], (~gv[6]) & 0xFFFFFFFF
        a_est, k1, e_key, ok, _ = self._k1(kmx, cfg)
        r = np.zeros((), dtype=_native.PRESCALE_RESULT_DTYPE)
        nnz = total_points - zeros
        r["a_max"] = r["p_tau"] = np.nan
        r["flags"], r["nnz"] = 4, nnz
        assert nnz > 0, "the CPU stand-in does not model all-zero images"
        if ok:
            r_lo = math.floor((nnz - 1) * (cfg.tau / 100.0))
            k = min(max(k1, cfg.k_min), cfg.k_max)
            e_mu = (mn >> 23) - 127
            if (32 * small <= r_lo and not rep and abs(k) <= 100 and lo >= -90 and hi <= 90 and lo + k >= -90
                    and hi + k <= 90 and e_mu >= -100 and e_mu + k >= -100 and e_key // 2 + k <= 100):
                r["a_max"], r["k1"], r["k2"], r["k"], r["flags"] = a_est, k1, -2**31, k, 8
        return r
