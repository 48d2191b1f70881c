"""Multi-GPU paths of the MX-FFT2; one process per GPU.

* Batches (C2/C3/C4): images are independent and each BASELINE image is its
  own prescale segment, so ranks take contiguous slices (`shard_range`) and
  run the single-GPU pipeline -- no collective on the data path.
* One very large image (C5, 16384^2): rank r owns rows [r*N/G, (r+1)*N/G).
  - The prescale is GLOBAL over the image (mri.py:88), built
    from device primitives plus collectives (`compute_prescale_global`):
    1. a sampled bracket from all ranks' keys (all_gather);
    2. one streaming count per rank (all_reduce SUM);
    3. the exact magnitudes of the few bracket candidates (all_gather);
    4. the peak (all_reduce MAX).
  - The 2-D transform (`fft2_slab`) runs the reference's rows-then-columns
    order (fftcore.py:351-353) as row passes on slabs with an all-to-all
    transpose between them.  x 2^k and 2^-k (and 1/N^2) are fused into the
    first and last row pass (mxfft_fft_rows_scaled).

Compute goes through `CudaOps` (the C-ABI kernels).  The communicator is a
torch.distributed process group: NCCL for CUDA tensors; gloo works too.
The tests drive the same orchestration on CPU with gloo, using a backend
built from the oracle (tests/cpu_ops.py).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native
from .errors import InvalidValue, UnsupportedSize
from .prescale import PrescaleConfig, PrescaleResult, k_from_stats

__all__ = ["shard_range", "Comm", "CudaOps", "compute_prescale_global", "prescale_fold_slab", "fft2_slab",
           "pipeline_slab"]


def shard_range(n_items: int, rank: int, world: int):
    """Contiguous [start, stop) of n_items for `rank` (the first n % world ranks take one more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class Comm:
    """The collectives the multi-GPU paths need, over a torch.distributed group
    (None = a single process: every collective is the identity)."""

    def __init__(self, group=None, enabled=None):
        import torch.distributed as dist

        self.dist = dist
        self.on = dist.is_available() and dist.is_initialized() if enabled is None else enabled
        self.group = group
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0

    def sum_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t

    def max_(self, t):
        if self.world > 1:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def all_gather_cat(self, t):
        """Concatenate 1-D tensors of (possibly) different lengths from all ranks."""
        import torch

        if self.world == 1:
            return t
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        m = max(sizes)
        pad = torch.zeros(m, dtype=t.dtype, device=t.device)
        pad[: t.numel()] = t
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return torch.cat([p[:s] for p, s in zip(parts, sizes)])

    def all_to_all(self, out, inp):
        if self.world == 1:
            out.copy_(inp)
        else:
            self.dist.all_to_all_single(out, inp, group=self.group)
        return out


class CudaOps:
    """The device primitives of the multi-rank paths, through the C-ABI."""

    def rows(self, x, plan, inverse: bool, exp_in: int = 0, exp_out: int = 0):
        import torch

        y = torch.empty_like(x)
        _native.check(_native.lib().mxfft_fft_rows_scaled(plan.handle, x.data_ptr(), y.data_ptr(),
                                                          x.numel() // plan.n, int(inverse), int(exp_in),
                                                          int(exp_out), _native.stream_handle()))
        return y

    def rows_seg(self, recv, plan, inverse: bool, exp_in: int = 0, exp_out: int = 0):
        """Row pass reading its lines straight from an all-to-all receive buffer
        (G, R, R): line c = recv[0][c] | recv[1][c] | ... (mxfft_fft_rows_seg) --
        no permute copy between the exchange and the pass."""
        import torch

        G, R, _ = recv.shape
        y = torch.empty((R, G * R), dtype=recv.dtype, device=recv.device)
        _native.check(_native.lib().mxfft_fft_rows_seg(plan.handle, recv.data_ptr(), y.data_ptr(), R, int(inverse),
                                                       int(exp_in), int(exp_out), R, _native.stream_handle()))
        return y

    def rows_evidence(self, x, plan, inverse: bool = False):
        """The first row pass on the unscaled input plus the evidence words of
        the folded prescale (mxfft_fft_rows_evidence) -> (rows, words)."""
        import torch

        L = _native.lib()
        y = torch.empty_like(x)
        nb = int(L.mxfft_fold_words_bytes(x.numel()))
        words = torch.empty(max(nb, 1), dtype=torch.uint8, device=x.device)
        _native.check(L.mxfft_fft_rows_evidence(plan.handle, x.data_ptr(), y.data_ptr(), x.numel() // plan.n,
                                                int(inverse), words.data_ptr(), nb, _native.stream_handle()))
        return y, words

    def fold_reduce(self, words, npoints: int, cfg: PrescaleConfig, step: int, g=None):
        """One reduction step of the folded prescale over this rank's words;
        g: int32 tensor of 8 words (bit patterns of uint32), created by step 0."""
        import torch

        if g is None:
            g = torch.empty(8, dtype=torch.int32, device=words.device)
        c = cfg.as_c()
        _native.check(_native.lib().mxfft_fold_reduce(words.data_ptr(), npoints, ctypes.byref(c), step, g.data_ptr(),
                                                      _native.stream_handle()))
        return g

    def fold_finish(self, g, total_points: int, cfg: PrescaleConfig):
        """-> the result row (numpy record: k, k1, flags, a_max, ...) from the combined words."""
        import torch

        from .prescale import decode_results

        res = torch.empty((1, _native.PRESCALE_RESULT_DTYPE.itemsize), dtype=torch.uint8, device=g.device)
        k = torch.empty(1, dtype=torch.int32, device=g.device)
        c = cfg.as_c()
        _native.check(_native.lib().mxfft_fold_finish(g.data_ptr(), total_points, ctypes.byref(c), res.data_ptr(),
                                                      k.data_ptr(), _native.stream_handle()))
        return decode_results(res)[0]  # (synchronizes: the one read-back of the folded prescale)

    def sample_keys(self, x, nsamples: int):
        import torch

        keys = torch.empty(nsamples, dtype=torch.float32, device=x.device)
        _native.check(_native.lib().mxfft_prescale_sample_keys(x.data_ptr(), x.numel(), nsamples,
                                                               keys.data_ptr(), _native.stream_handle()))
        return keys

    def count_range(self, x, lo: float, hi: float, top: float, cand_cap: int, top_cap: int):
        """-> (nnz, below, ncand, ntop, flags) and the candidate / top values (complex64)."""
        import torch

        state = torch.zeros(40, dtype=torch.uint8, device=x.device)
        cand = torch.empty(max(cand_cap, 1), dtype=torch.complex64, device=x.device)
        topb = torch.empty(max(top_cap, 1), dtype=torch.complex64, device=x.device)
        _native.check(_native.lib().mxfft_prescale_count_range(
            x.data_ptr(), x.numel(), ctypes.c_float(lo), ctypes.c_float(hi), ctypes.c_float(top),
            state.data_ptr(), cand.data_ptr(), cand_cap, topb.data_ptr(), top_cap, _native.stream_handle()))
        s = state.cpu().numpy().tobytes()
        nnz = int(np.frombuffer(s, dtype="<u8", count=1, offset=16)[0])
        below, ncand, ntop, flags = (int(v) for v in np.frombuffer(s, dtype="<u4", count=4, offset=24))
        return (nnz, below, ncand, ntop, flags), cand[: min(ncand, cand_cap)], topb[: min(ntop, top_cap)]

    def block_transpose(self, a, g: int):
        """(R, G*R) slab -> (G, R, R) send buffer, block j = (a[:, jR:(j+1)R])^T
        (mxfft_transpose_c64_strided; torch's copy for R not a multiple of 64)."""
        import torch

        R = a.shape[0]
        out = torch.empty((g, R, R), dtype=a.dtype, device=a.device)
        if R % 64 or a.dtype != torch.complex64:
            out.copy_(a.reshape(R, g, R).permute(1, 2, 0))
            return out
        _native.check(_native.lib().mxfft_transpose_c64_strided(a.data_ptr(), a.shape[1], R, out.data_ptr(), g, R,
                                                                _native.stream_handle()))
        return out

    def cabs(self, z):
        import torch

        out = torch.empty(z.numel(), dtype=torch.float64, device=z.device)
        _native.check(_native.lib().mxfft_cabs(z.data_ptr(), 0, z.numel(), out.data_ptr(),
                                               _native.stream_handle()))
        return out


def _bracket_dev(keys_sorted, n: int, q: float, widen: float):
    """Sample ranks around the tau-quantile -> FP32 key bracket [lo, hi] and the
    peak threshold (the same rule as the fused kernel, k_ps_fused), from a
    sorted torch tensor (any device) whose first n entries are finite; only the
    three order statistics it needs are read back."""
    import torch

    if n == 0:
        return np.float32(0.0), np.float32(np.inf), np.float32(0.0), n
    rs = (n - 1) * q
    d = int((8 + 4.0 * math.sqrt(rs + 1.0)) * widen)
    ilo, ihi = int(math.floor(rs)) - d, int(math.ceil(rs)) + 1 + d
    idx = torch.tensor([max(ilo, 0), min(ihi, n - 1), n - 1], dtype=torch.int64, device=keys_sorted.device)
    v = keys_sorted[idx].cpu().numpy().astype(np.float32)
    f32 = np.float32
    lo = f32(0.0) if ilo <= 0 else f32(v[0]) * f32(1 - 2.0**-20)
    hi = f32(np.inf) if ihi >= n else f32(v[1]) * f32(1 + 2.0**-20)
    top = f32(v[2]) * f32(1 - 2.0**-20)
    return lo, hi, top, n


def compute_prescale_global(x_local, cfg: PrescaleConfig, comm: Comm = None, ops=None,
                            nsamples: int = 1 << 18) -> PrescaleResult:
    """compute_prescale (prescale.py:61-73) over ONE segment whose points are
    split across the ranks of `comm` (each passes its complex64 share, a
    multiple of 4 points).  Exact: the same a_max, p_tau and k as the reference
    on the whole segment.  Synchronizes the host (it returns Python scalars)."""
    import torch

    comm = comm or Comm(enabled=False)
    ops = ops or CudaOps()
    x = x_local.reshape(-1)
    if x.dtype != torch.complex64:
        raise TypeError("global statistics take complex64 data")
    npts = x.numel()
    q = cfg.tau / 100.0
    s_local = min(max(4, (nsamples // comm.world) // 4 * 4), npts // 4 * 4)
    keys = torch.sort(comm.all_gather_cat(ops.sample_keys(x, s_local))).values
    # the sorted sample stays where it is: only the few order statistics and
    # bracket counts the host needs are read back (not the whole sample)
    n_fin = int(torch.isfinite(keys).sum())
    dev = x.device
    for widen in (1.0, 4.0, 32.0, None):
        if widen is None:  # last resort: every nonzero point is a candidate
            lo, hi, top, nsamp = np.float32(0.0), np.float32(np.inf), np.float32(0.0), 0
        else:
            lo, hi, top, nsamp = _bracket_dev(keys, n_fin, q, widen)
        if nsamp == 0:
            cand_cap, top_cap = npts, npts
        else:
            fin = keys[:nsamp]
            edges = torch.tensor([float(hi), float(lo)], dtype=fin.dtype, device=fin.device)
            above = int(torch.searchsorted(fin, edges[:1], right=True).item())
            below_lo = int(torch.searchsorted(fin, edges[1:], right=False).item())
            f = (min(nsamp, above) - below_lo) / nsamp
            cand_cap = min(npts, int(npts * f * 2) + 65536)
            top_cap = min(npts, int(4 * npts / nsamp) + 4096)
        (nnz, below, ncand, ntop, flags), cand, topb = ops.count_range(x, float(lo), float(hi), float(top),
                                                                       cand_cap, top_cap)
        tot = torch.tensor([nnz, below, ncand, ntop, flags, int(ncand > cand_cap or ntop > top_cap)],
                           dtype=torch.int64, device=dev)
        nnz, below, ncand, ntop, flags, overflow = (int(v) for v in comm.sum_(tot).cpu())
        if flags:
            if not bool(comm.max_(torch.tensor([int(not torch.isfinite(x).all())], device=dev)).item()):
                raise UnsupportedSize("magnitudes outside [2^-60, 2^60] need the single-segment exact "
                                      "statistics (prescale_stats_device)")
            raise InvalidValue("non-finite input to prescale")
        if nnz == 0:
            a_max = p_tau = 0.0
            break
        virt = (nnz - 1) * q
        if virt >= nnz - 1:
            r_lo = r_hi = nnz - 1
            gamma = virt + 1.0
        else:
            r_lo = int(math.floor(virt))
            r_hi = r_lo + 1
            gamma = virt - r_lo
        if overflow or ntop < 1 or not (below <= r_lo and r_hi < below + ncand):
            continue  # widen the bracket
        mags = torch.sort(comm.all_gather_cat(ops.cabs(cand))).values
        vlo, vhi = float(mags[r_lo - below].item()), float(mags[r_hi - below].item())
        # points outside the bracket must order strictly on their side: the
        # picks clear the bracket's key edges by more than the FP32 key rounding
        if lo > 0 and not (vlo * vlo > float(lo) * (1.0 + 2.0**-18)):
            continue
        if np.isfinite(hi) and not (vhi * vhi < float(hi) * (1.0 - 2.0**-18)):
            continue
        tmax = ops.cabs(topb)
        a_max = float(comm.max_(tmax.max().reshape(1) if tmax.numel() else
                                torch.zeros(1, dtype=torch.float64, device=dev)).item())
        diff = vhi - vlo
        p_tau = vhi - diff * (1.0 - gamma) if gamma >= 0.5 else vlo + diff * gamma
        break
    else:  # pragma: no cover - the last attempt always settles
        raise RuntimeError("global prescale statistics did not settle")
    k, k1, k2 = k_from_stats(a_max, p_tau, cfg)
    return PrescaleResult(k=k, a_max=a_max, p_tau=p_tau, k1=k1, k2=k2)


def _exchange(a, comm: Comm, ops):
    """(R, N) = this rank's rows of A  ->  the receive buffer (G, R, R) of one
    all-to-all of R x R blocks: recv[i][c][r] =
    A[i R + r][me R + c], i.e. row c of this rank's rows of A^T is the
    concatenation recv[0][c] | recv[1][c] | ...  The sender transposes each
    block on the way into the send buffer (one kernel); the next row pass
    reads the receive layout directly (CudaOps.rows_seg)."""
    import torch

    G = comm.world
    send = ops.block_transpose(a, G)  # [j][c][r] = A[me*R + r][j*R + c]
    recv = torch.empty_like(send)
    comm.all_to_all(recv, send)
    return recv


def _transpose_slabs(a, comm: Comm, ops):
    """(R, N) = this rank's rows of A  ->  (R, N) = this rank's rows of A^T,
    materialised (only for a restored output layout)."""
    R, N = a.shape
    recv = _exchange(a, comm, ops)
    return recv.permute(1, 0, 2).reshape(R, N).contiguous()  # [c][i*R + r] = A^T[me*R + c][i*R + r]


def fft2_slab(x_slab, plan, mode: str = "forward", comm: Comm = None, ops=None, k: int = 0,
              restore: bool = True, first_pass=None):
    """fft_2d (fftcore.py:344-353) of one N x N image whose rows are split across
    the ranks of `comm`; x_slab is this rank's (N/G, N) complex64 row slab.
    mode: "forward" | "inverse" | "roundtrip" (forward, inverse, x 1/N^2).
    k: prescale exponent, x 2^k on the first load and 2^-k on the last store.
    Returns this rank's rows of the result (restore=True), else its rows of
    the transposed result (one all-to-all fewer).
    first_pass: the first row pass's output when it already ran on the
    UNSCALED slab (the folded prescale, pipeline_slab): x 2^k then moves to the
    load of the second pass, which is exact."""
    comm = comm or Comm(enabled=False)
    ops = ops or CudaOps()
    N = plan.n
    G = comm.world
    if N % G:
        raise UnsupportedSize(f"{N} rows do not split over {G} ranks")
    if tuple(x_slab.shape) != (N // G, N):
        raise UnsupportedSize(f"expected a ({N // G}, {N}) slab, got {tuple(x_slab.shape)}")
    dirs = {"forward": (False, False), "inverse": (True, True),
            "roundtrip": (False, False, True, True)}[mode]
    out_exp = -k - (2 * plan.stages if mode == "roundtrip" else 0)
    y = x_slab.contiguous()
    k_at = 0 if first_pass is None else 1  # the pass whose load applies 2^k
    for i, inv in enumerate(dirs):
        last = i == len(dirs) - 1
        e_in, e_out = (k if i == k_at else 0), (out_exp if last else 0)
        if i == 0 and first_pass is not None:
            y = first_pass
        elif i == 0:
            y = ops.rows(y, plan, inv, exp_in=e_in, exp_out=e_out)
        elif hasattr(ops, "rows_seg"):
            # every later pass works on the rows of the previous result's
            # transpose, read straight from the all-to-all receive buffer
            y = ops.rows_seg(_exchange(y, comm, ops), plan, inv, exp_in=e_in, exp_out=e_out)
        else:
            y = ops.rows(_transpose_slabs(y, comm, ops), plan, inv, exp_in=e_in, exp_out=e_out)
    return _transpose_slabs(y, comm, ops) if restore else y


def _u32(g):
    """int32 bit patterns -> int64 values in [0, 2^32) (all-reduce MAX / SUM on unsigned words)."""
    import torch

    return g.to(torch.int64) & 0xFFFFFFFF


def _i32(a):
    """int64 values in [0, 2^32) -> the int32 tensor with the same bit patterns."""
    import torch

    return (((a + 2**31) % 2**32) - 2**31).to(torch.int32)


def prescale_fold_slab(x_slab, plan, cfg: PrescaleConfig, comm: Comm, ops):
    """compute_prescale (prescale.py:61-73) over the whole image FOLDED into the
    first row pass of this rank's slab: the pass runs unscaled and gathers the
    evidence (mxfft_fft_rows_evidence); two small all-reduces combine it (MAX
    of the peak key / exponent range, then SUM of the counts under the global
    threshold) and every rank settles the same k (mxfft_fold_finish) with one
    read-back.  Returns (first-pass rows, result row); row["flags"] & 4: the
    proofs declined and the caller takes the statistics path."""
    import torch

    npts = x_slab.numel()
    y1, words = ops.rows_evidence(x_slab, plan, False)
    g = ops.fold_reduce(words, npts, cfg, 0)
    if comm.world > 1:
        a = _u32(g[:4])
        comm.max_(a)
        g[:4] = _i32(a)
    ops.fold_reduce(words, npts, cfg, 1, g)
    if comm.world > 1:
        cnt, mn = _u32(g[4:6]), _u32(g[6:7])
        comm.sum_(cnt)
        comm.max_(mn)
        g[4:6] = _i32(cnt)
        g[6:7] = _i32(mn)
    return y1, ops.fold_finish(g, plan.n * plan.n, cfg)  # (the slabs partition one n x n image)


def pipeline_slab(x_slab, plan, cfg: PrescaleConfig, roundtrip: bool, comm: Comm = None, ops=None,
                  fold=None, restore: bool = True):
    """The C5 pipeline on row slabs: global prescale, then the 2-D transform
    with the scalings fused (forward_pipeline / roundtrip_pipeline,
    mri.py:84-107, for one coil).  Returns (this rank's rows of the output, the
    prescale result).

    fold (default: on when the backend provides it and n = 16384): the
    prescale rides on the first row pass (prescale_fold_slab) -- no statistics
    pass over the slab, one host read-back instead of several.  If its proofs
    decline, the statistics path below runs instead; results are identical."""
    comm = comm or Comm(enabled=False)
    ops = ops or CudaOps()
    mode = "roundtrip" if roundtrip else "forward"
    use_fold = (hasattr(ops, "rows_evidence") and plan.n == 16384) if fold is None else fold
    if use_fold:
        y1, row = prescale_fold_slab(x_slab, plan, cfg, comm, ops)
        if not int(row["flags"]) & 4:
            res = PrescaleResult(k=int(row["k"]), a_max=float(row["a_max"]), p_tau=float(row["p_tau"]),
                                 k1=int(row["k1"]), k2=int(row["k2"]))
            y = fft2_slab(x_slab, plan, mode, comm, ops, k=res.k, restore=restore, first_pass=y1)
            return y, res
        del y1
    res = compute_prescale_global(x_slab, cfg, comm, ops)
    y = fft2_slab(x_slab, plan, mode, comm, ops, k=res.k, restore=restore)
    return y, res
