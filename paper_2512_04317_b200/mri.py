"""MRI-style pipelines on the GPU: prescale -> MX-FFT2 (-> inverse) -> undo -> RSS.

Public surface of pkg/src/mxfft/mri.py:35-107 (ComplexGrid, RssImage, rss,
forward_pipeline, roundtrip_pipeline).  One coil stack shares one global
prescale exponent (mri.py:88, mri.py:98); every coil is transformed
independently.  On the device the whole pipeline is:

  mxfft_prescale_stats (k on device, no host sync)
  mxfft_fft2 (x*2^k fused into the first load, 2^-k [and 1/N^2] into the last store)
  mxfft_rss (|T_c| summed over coils, numpy-exact magnitude)

The batched entry points (*_device) take (B, N, N) complex64 CUDA tensors and
give each image its own prescale (C = 1 stacks) -- the BASELINE workloads.
"""

from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np

from . import _native
from .errors import InvalidValue, ShapeError
from .fftcore import FftPlan, fft2_device
from .prescale import (PrescaleConfig, decode_results, k_from_stats, prescale_stats_device)

KSPACE = "kspace"
IMAGE = "image"


@dataclasses.dataclass(frozen=True)
class ComplexGrid:
    """(coils, n, n) complex128 samples tagged "kspace" or "image"."""

    data: np.ndarray
    domain: str

    def __post_init__(self):
        d = np.asarray(self.data, dtype=np.complex128)
        if d.ndim != 3 or d.shape[1] != d.shape[2]:
            raise ShapeError("grid data must be (coils, n, n)")
        if self.domain not in (KSPACE, IMAGE):
            raise InvalidValue(f"unknown domain tag {self.domain!r}")
        if not np.isfinite(d).all():
            raise InvalidValue("non-finite grid data")
        object.__setattr__(self, "data", d)

    @property
    def coils(self) -> int:
        return self.data.shape[0]

    @property
    def n(self) -> int:
        return self.data.shape[1]


@dataclasses.dataclass(frozen=True)
class RssImage:
    pixels: np.ndarray  # (n, n) nonnegative FP64

    @property
    def n(self) -> int:
        return self.pixels.shape[0]


def rss_device(x, coils: int = 1):
    """RSS of a CUDA complex tensor (groups*coils, ...) -> CUDA float64 (groups, ...)."""
    import torch

    x = x.contiguous()
    npix = x[0].numel()
    groups = x.shape[0] // coils
    out = torch.empty((groups,) + tuple(x.shape[1:]), dtype=torch.float64, device=x.device)
    _native.check(_native.lib().mxfft_rss(x.data_ptr(), int(x.dtype == torch.complex128), groups,
                                          coils, npix, out.data_ptr(), _native.stream_handle()))
    return out


def rss(images) -> RssImage:
    """sqrt(sum_c |T_c|^2) per pixel (coil combine)."""
    import torch

    if isinstance(images, ComplexGrid):
        stack = images.data
    else:
        arrs = [np.asarray(a, dtype=np.complex128) for a in images]
        if not arrs:
            raise ShapeError("need at least one coil")
        if any(a.shape != arrs[0].shape for a in arrs):
            raise ShapeError("coil images must share one shape")
        stack = np.stack(arrs)
    t = torch.from_numpy(np.ascontiguousarray(stack)).cuda()
    return RssImage(rss_device(t, coils=stack.shape[0])[0].cpu().numpy())


# ---------------------------------------------------------------------------
# batched, device-resident pipelines (one prescale per image)
# ---------------------------------------------------------------------------
# pipeline_device's default for n = 128 images: the statistics kernel + four
# line passes (measured faster on B200: 1.08 vs 1.25 ms for C4)
# or, with MXFFT_FUSED=1, the fused one-image-per-CTA kernel
# (mxfft_pipeline_fused).  Results are identical either way.
FUSED = os.environ.get("MXFFT_FUSED", "0") == "1"
# n = 128 / 256 / 512: compute_prescale folded into the first transform pass
# (mxfft_pipeline_folded: no standalone statistics read of x).  Stacks the
# in-kernel proofs cannot settle come back with flag bit 2 and are re-run by
# pipeline_resolve through the statistics kernels.  MXFFT_FOLD=0 turns it off.
FOLD = os.environ.get("MXFFT_FOLD", "1") == "1"
# (plan, config) pairs for which pipeline_resolve found the fold unproductive (more than a
# quarter of a call's stacks unsettled, e.g. a configuration in which k2 wins): later default calls
# run the statistics kernels directly instead of transforming twice.  fold=True still forces it.
_FOLD_UNPRODUCTIVE = set()


def fused_pipeline_supported(plan: FftPlan, coils: int = 1) -> bool:
    """True when pipeline_device runs the whole per-image pipeline as one fused
    kernel (one 128 x 128 image per CTA, every stage in shared memory; the
    BASELINE configs[3] workload)."""
    if coils != 1 or plan.mode.kind != "mx":
        return False
    return bool(_native.load().mxfft_pipeline_fused_supported(plan.handle))


def folded_pipeline_supported(plan: FftPlan) -> bool:
    """True when pipeline_device can fold the prescale statistics into the first
    transform pass (n = 128 / 256 / 512, hardware MX formats, B in {16, 32, 64})."""
    if plan.mode.kind != "mx":
        return False
    return bool(_native.load().mxfft_pipeline_folded_supported(plan.handle))


def pipeline_device(x, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool, coils: int = 1,
                    out=None, k=None, res=None, fused=None, fold=None):
    """x: CUDA complex64 (B*coils, N, N).  Stacks of `coils` consecutive images
    share one prescale (C = 1: per image).  Returns (out complex64, k int32 (B,),
    stats uint8 (B, 40)) without synchronizing.

    The statistics rows carry the reference's error cases as flags (the host
    is not consulted on this path): bit 0 = non-finite input (the reference
    raises InvalidValue), bit 1 = a log2 within a few ulps of a rounding
    boundary (k must be confirmed with the host's log2).  pipeline_resolve
    turns them into the reference's behaviour after the fact; pipeline_host
    calls it on every step.

    fold (default: the module's FOLD, on): for n = 128 / 256 / 512 the
    statistics ride on the first transform pass (mxfft_pipeline_folded).  Rows
    it settles carry flag bit 3 (k exact; a_max approximate, p_tau not
    evaluated); a stack it cannot settle carries bit 2, its output is
    unspecified until pipeline_resolve has re-run it.  fold=False always runs
    the statistics kernels first (full rows)."""
    if x.dim() != 3 or coils < 1 or x.shape[0] % coils:
        raise ShapeError(f"batch of {x.shape[0]} images is not a whole number of {coils}-coil stacks")
    n = plan.n
    nstack = x.shape[0] // coils
    for t, name in ((k, "k"), (res, "res")):
        if t is not None and t.shape[0] < nstack:
            raise ShapeError(f"{name} buffer holds {t.shape[0]} stacks, need {nstack}")
    use_fused = FUSED if fused is None else fused
    if use_fused and fused_pipeline_supported(plan, coils) and (out is None or out.data_ptr() != x.data_ptr()):
        import torch

        if x.dtype != torch.complex64 or not x.is_cuda:
            raise TypeError("expected a CUDA complex64 tensor")
        x = x.contiguous()
        y = out if out is not None else torch.empty_like(x)
        res = res if res is not None else torch.empty((nstack, _native.PRESCALE_RESULT_DTYPE.itemsize),
                                                      dtype=torch.uint8, device=x.device)
        k = k if k is not None else torch.empty(nstack, dtype=torch.int32, device=x.device)
        c = cfg.as_c()
        _native.check(_native.lib().mxfft_pipeline_fused(plan.handle, x.data_ptr(), y.data_ptr(), nstack,
                                                         int(bool(roundtrip)), ctypes.byref(c), res.data_ptr(),
                                                         k.data_ptr(), _native.stream_handle()))
        return y, k, res
    use_fold = (FOLD and (id(plan), repr(cfg)) not in _FOLD_UNPRODUCTIVE) if fold is None else fold
    if (use_fold and not use_fused and x.is_cuda and nstack > 0 and folded_pipeline_supported(plan)
            and (out is None or out.data_ptr() != x.data_ptr())):
        import torch

        if x.dtype != torch.complex64:
            raise TypeError("expected a CUDA complex64 tensor")
        x = x.contiguous()
        y = out if out is not None else torch.empty_like(x)
        res = res if res is not None else torch.empty((nstack, _native.PRESCALE_RESULT_DTYPE.itemsize),
                                                      dtype=torch.uint8, device=x.device)
        k = k if k is not None else torch.empty(nstack, dtype=torch.int32, device=x.device)
        L = _native.lib()
        need = int(L.mxfft_pipeline_folded_workspace_bytes(plan.handle, x.shape[0], coils))
        ws = torch.empty(need, dtype=torch.uint8, device=x.device)
        c = cfg.as_c()
        _native.check(L.mxfft_pipeline_folded(plan.handle, x.data_ptr(), y.data_ptr(), x.shape[0], coils,
                                              int(bool(roundtrip)), ctypes.byref(c), res.data_ptr(), k.data_ptr(),
                                              ws.data_ptr(), need, _native.stream_handle()))
        return y, k, res
    res, k = prescale_stats_device(x, nstack, coils * n * n, cfg, k_out=k, res_out=res)
    y = fft2_device(x, plan, "roundtrip" if roundtrip else "forward", k=k, k_group=coils, out=out)
    return y, k, res


def pipeline_resolve(x, y, k, res, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool, coils: int = 1):
    """Settle the flags of a pipeline_device call (synchronizes): raise
    InvalidValue for a stack with non-finite input (prescale.py:63-64), and
    re-derive k with the host's log2 (= the reference's math.log2) for stacks
    whose device log2 sat on a rounding boundary, re-running those stacks when
    k changes.  Returns the number of stacks re-run (0 for real data)."""
    import torch

    r = decode_results(res)
    redo = 0
    unsettled = np.nonzero(r["flags"] & 4)[0]
    if unsettled.size:
        # the folded pipeline could not prove k for these stacks: statistics kernels + standard
        # passes on each run of consecutive stacks, then their rows are looked at like any other
        runs = np.split(unsettled, np.nonzero(np.diff(unsettled) != 1)[0] + 1)
        for run in runs:
            a, b = int(run[0]), int(run[-1]) + 1
            sl = slice(a * coils, b * coils)
            pipeline_device(x[sl], plan, cfg, roundtrip, coils=coils, out=y[sl], k=k[a:b], res=res[a:b],
                            fused=False, fold=False)
        redo += int(unsettled.size)
        if 4 * unsettled.size > r.size:
            _FOLD_UNPRODUCTIVE.add((id(plan), repr(cfg)))
        r = decode_results(res)
    bad = np.nonzero(r["flags"] & 1)[0]
    if bad.size:
        raise InvalidValue(f"non-finite input to prescale (stacks {bad[:8].tolist()})")
    for i in np.nonzero(r["flags"] & 2)[0]:
        kh, _, _ = k_from_stats(float(r["a_max"][i]), float(r["p_tau"][i]), cfg)
        if kh == int(r["k"][i]):
            continue
        k[i] = kh
        sl = slice(int(i) * coils, (int(i) + 1) * coils)
        fft2_device(x[sl], plan, "roundtrip" if roundtrip else "forward", k=k[i:i + 1], k_group=coils,
                    out=y[sl])
        redo += 1
    if redo:
        torch.cuda.current_stream().synchronize()
    return redo


_HOST_PIPE = {}  # per device: the three streams of pipeline_host

# device staging budget of pipeline_host: batches up to this size get whole-batch
# device buffers (no ring back-pressure between the copy streams and compute)
HOST_PIPE_DEVICE_BYTES = 16 << 30


def host_slices(nstack: int, chunks: int):
    """Slice sizes (in coil stacks) for pipeline_host: `chunks` slices with
    weights 1, 2, 4, ..., 4, 2, 1.  Nothing overlaps the first H2D, so it is
    short; after it, H2D and D2H run at the same rate, so a slice no larger than
    the lead the D2H stream starts with is ready (copied in and transformed) by
    the time the D2H stream reaches it.  Nothing overlaps the last slice's
    compute and D2H either, so the tail tapers the same way (measured on C2:
    3.48 -> 3.40 ms per step, tools/e2e_taper.py).  Sizes sum to nstack; none
    is empty."""
    chunks = max(1, min(chunks, nstack))
    w = [min(4, 2 ** i, 2 ** (chunks - 1 - i)) for i in range(chunks)]
    tot = float(sum(w))
    sizes = [max(1, int(nstack * wi / tot)) for wi in w]
    # hand the rounding remainder to the largest (middle) slices
    d = nstack - sum(sizes)
    order = sorted(range(chunks), key=lambda j: -w[j])
    j = 0
    while d != 0:
        k = order[j % chunks]
        if d > 0:
            sizes[k] += 1
            d -= 1
        elif sizes[k] > 1:
            sizes[k] -= 1
            d += 1
        j += 1
    return sizes


_HOST_GRAPHS = {}  # (device, buffers, shape, plan, cfg, ...) -> captured pipeline_host step
_HOST_GRAPHS_MAX = 4


def pipeline_host(x_host, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool, out_host=None,
                  coils: int = 1, chunks: int = 14, graph: bool = True):
    """pipeline_device for a batch in (pinned) host memory -- see
    _pipeline_host_eager for the slicing and stream overlap.

    With graph=True and pinned buffers, the whole step (every H2D slice, the
    kernels, every D2H slice, on three streams) is captured once per
    (buffers, shape, plan, cfg, roundtrip, coils, chunks) as a CUDA graph and
    replayed on later calls: the copies still run every call (the graph's
    memcpy nodes read and write the caller's host buffers at replay time), but
    the host no longer spends ~0.1 ms of Python per slice enqueueing them."""
    import torch

    if x_host.is_cuda or x_host.dtype != torch.complex64:
        raise TypeError("pipeline_host takes a host complex64 tensor")
    if out_host is None:
        out_host = torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory()
    if not (graph and x_host.is_pinned() and out_host.is_pinned() and x_host.shape[0] > 0
            and x_host.is_contiguous() and out_host.is_contiguous()):
        return _pipeline_host_eager(x_host, plan, cfg, roundtrip, out_host, coils, chunks)
    dev = torch.cuda.current_device()
    key = (dev, x_host.data_ptr(), out_host.data_ptr(), tuple(x_host.shape), id(plan), plan.n,
           repr(cfg), bool(roundtrip), int(coils), int(chunks), (id(plan), repr(cfg)) in _FOLD_UNPRODUCTIVE)
    ent = _HOST_GRAPHS.get(key)
    if ent is None or ent[1] is not plan:
        _pipeline_host_eager(x_host, plan, cfg, roundtrip, out_host, coils, chunks)  # warm-up
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        stats = []  # the captured statistics rows (graph-pool memory, rewritten by every replay)
        with torch.cuda.graph(g, stream=cs):
            _pipeline_host_eager(x_host, plan, cfg, roundtrip, out_host, coils, chunks, capture=True,
                                 stats=stats)
        if len(_HOST_GRAPHS) >= _HOST_GRAPHS_MAX:
            _HOST_GRAPHS.pop(next(iter(_HOST_GRAPHS)))
        ent = (g, plan, stats)
        _HOST_GRAPHS[key] = ent
    ent[0].replay()
    torch.cuda.current_stream().synchronize()
    _resolve_host(x_host, out_host, ent[2], plan, cfg, roundtrip, coils)
    return out_host


def _resolve_host(x_host, out_host, stats, plan, cfg, roundtrip, coils):
    """pipeline_resolve for pipeline_host: one small D2H of the statistics rows
    of every slice; stacks the folded pipeline left unsettled (flag bit 2) are
    redone from the host copy through the statistics kernels; InvalidValue for
    non-finite stacks; stacks whose k sat on a log2 rounding boundary are
    redone with the host's k (never for real data)."""
    import torch

    if not stats:
        return
    r = decode_results(torch.cat([t for t in stats])).copy()
    mode = "roundtrip" if roundtrip else "forward"
    if 4 * int((r["flags"] & 4 != 0).sum()) > r.size:
        _FOLD_UNPRODUCTIVE.add((id(plan), repr(cfg)))  # (pipeline_host then captures a new graph without the fold)
    for i in np.nonzero(r["flags"] & 4)[0]:
        # a stack the folded pipeline could not settle: statistics kernels + standard passes
        # from the host copy; its full row then goes through the checks below
        sl = slice(int(i) * coils, (int(i) + 1) * coils)
        xd = x_host[sl].cuda()
        y, _, rs = pipeline_device(xd, plan, cfg, roundtrip, coils=coils, fused=False, fold=False)
        r[i] = decode_results(rs)[0]
        if not int(r["flags"][i]) & 1:
            out_host[sl].copy_(y.cpu())
    bad = np.nonzero(r["flags"] & 1)[0]
    if bad.size:
        raise InvalidValue(f"non-finite input to prescale (stacks {bad[:8].tolist()})")
    for i in np.nonzero(r["flags"] & 2)[0]:
        kh, _, _ = k_from_stats(float(r["a_max"][i]), float(r["p_tau"][i]), cfg)
        if kh == int(r["k"][i]):
            continue
        sl = slice(int(i) * coils, (int(i) + 1) * coils)
        xd = x_host[sl].cuda()
        kd = torch.tensor([kh], dtype=torch.int32, device=xd.device)
        y = fft2_device(xd, plan, mode, k=kd, k_group=coils)
        out_host[sl].copy_(y.cpu())


def _pipeline_host_eager(x_host, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool, out_host=None,
                         coils: int = 1, chunks: int = 8, capture: bool = False, stats=None):
    """pipeline_device for a batch that lives in (pinned) host memory.

    The batch is cut into `chunks` slices of whole coil stacks (host_slices:
    a short first slice, then equal ones).  Three streams: slice i+1
    is copied in while slice i is transformed and slice i-1 is copied out (PCIe
    is full duplex).  Batches up to HOST_PIPE_DEVICE_BYTES are staged in
    whole-batch device buffers, so the H2D stream never waits for compute or
    D2H; larger batches cycle through two slice-sized buffers.
    x_host: CPU complex64 (B*coils, N, N), pinned for overlap.  Returns
    out_host (allocated pinned if None) once every copy has finished."""
    import torch

    if x_host.is_cuda or x_host.dtype != torch.complex64:
        raise TypeError("pipeline_host takes a host complex64 tensor")
    n = plan.n
    if x_host.dim() != 3 or coils < 1 or x_host.shape[0] % coils:
        raise ShapeError(f"batch of {x_host.shape[0]} images is not a whole number of {coils}-coil stacks")
    nstack = x_host.shape[0] // coils
    if out_host is None:
        out_host = torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory()
    if nstack == 0:
        return out_host
    own_stats = stats is None
    if own_stats:
        stats = []
    sizes = host_slices(nstack, chunks)
    dev = torch.device("cuda", torch.cuda.current_device())
    key = str(dev)
    if key not in _HOST_PIPE:
        _HOST_PIPE[key] = [torch.cuda.Stream(dev) for _ in range(3)]
    s_in, s_cmp, s_out = _HOST_PIPE[key]
    cur = torch.cuda.current_stream(dev)
    whole = 2 * x_host.numel() * 8 <= HOST_PIPE_DEVICE_BYTES
    if whole:
        xb = [torch.empty(x_host.shape, dtype=torch.complex64, device=dev)]
        yb = [torch.empty(x_host.shape, dtype=torch.complex64, device=dev)]
        kb = [torch.empty(nstack, dtype=torch.int32, device=dev)]
    else:
        per = max(sizes) * coils
        xb = [torch.empty((per, n, n), dtype=torch.complex64, device=dev) for _ in range(2)]
        yb = [torch.empty((per, n, n), dtype=torch.complex64, device=dev) for _ in range(2)]
        kb = [torch.empty(per // coils, dtype=torch.int32, device=dev) for _ in range(2)]
    nb = len(xb)
    ev_cmp = [None] * nb
    ev_out = [None] * nb
    for s in (s_in, s_cmp, s_out):
        s.wait_stream(cur)  # buffers were allocated on the current stream
    start = 0
    for i, sz in enumerate(sizes):
        b = i % nb
        m = sz * coils
        if whole:
            xs, ys, ks = xb[0][start:start + m], yb[0][start:start + m], kb[0][start // coils:start // coils + sz]
        else:
            xs, ys, ks = xb[b][:m], yb[b][:m], kb[b][:sz]
            if ev_cmp[b] is not None:
                s_in.wait_event(ev_cmp[b])  # slice i-2 no longer reads xb[b]
        with torch.cuda.stream(s_in):
            xs.copy_(x_host[start:start + m], non_blocking=True)
            e_in = torch.cuda.Event()
            e_in.record(s_in)
        s_cmp.wait_event(e_in)
        if not whole and ev_out[b] is not None:
            s_cmp.wait_event(ev_out[b])  # slice i-2 has left yb[b]
        with torch.cuda.stream(s_cmp):
            _, _, rs = pipeline_device(xs, plan, cfg, roundtrip, coils=coils, out=ys, k=ks)
            stats.append(rs)
            ev_cmp[b] = torch.cuda.Event()
            ev_cmp[b].record(s_cmp)
        s_out.wait_event(ev_cmp[b])
        with torch.cuda.stream(s_out):
            out_host[start:start + m].copy_(ys, non_blocking=True)
            ev_out[b] = torch.cuda.Event()
            ev_out[b].record(s_out)
        start += m
    for t in xb + yb + kb:
        for s in (s_in, s_cmp, s_out):
            t.record_stream(s)
    for s in (s_in, s_cmp, s_out):
        cur.wait_stream(s)
    if not capture:
        s_out.synchronize()
        s_cmp.synchronize()
        if own_stats:
            _resolve_host(x_host, out_host, stats, plan, cfg, roundtrip, coils)
    return out_host


def _run_grid(grid: ComplexGrid, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool) -> RssImage:
    """The reference's order of operations (mri.py:84-107), on the GPU:
    statistics on the caller's FP64 values (prescale.py:61-73) -> x * 2^k in
    FP64, cast to complex64 (prescale.py:83, fftcore.py:262) -> FP32 MX
    transforms -> x 1/N^2 and x 2^-k in FP64 -> RSS.  So results match the
    reference even where the scaled values leave FP32's normal range."""
    import torch

    x128 = torch.from_numpy(np.ascontiguousarray(grid.data)).cuda()
    res, k = prescale_stats_device(x128, 1, x128.numel(), cfg)
    r = decode_results(res)[0]
    if int(r["flags"]) & 1:
        raise InvalidValue("non-finite input to prescale")
    if int(r["flags"]) & 2:  # k near a log2 rounding boundary: decide on the host
        kh, _, _ = k_from_stats(float(r["a_max"]), float(r["p_tau"]), cfg)
        if kh != int(r["k"]):
            k = torch.tensor([kh], dtype=torch.int32, device=x128.device)
    L = _native.lib()
    x = torch.empty(x128.shape, dtype=torch.complex64, device=x128.device)
    _native.check(L.mxfft_prescale_apply_c128(x128.data_ptr(), x.data_ptr(), 1, x128.numel(), k.data_ptr(),
                                              _native.stream_handle()))
    y = fft2_device(x, plan, "forward")
    if roundtrip:
        y = fft2_device(y, plan, "inverse", out=y)
    n = grid.n
    out = torch.empty((1, n, n), dtype=torch.float64, device=x.device)
    econst = -2 * (plan.n.bit_length() - 1) if roundtrip else 0
    _native.check(L.mxfft_rss_scaled(y.data_ptr(), 0, 1, grid.coils, n * n, k.data_ptr(), -1, econst,
                                     out.data_ptr(), _native.stream_handle()))
    return RssImage(out[0].cpu().numpy())


def forward_pipeline(kspace: ComplexGrid, plan: FftPlan, cfg: PrescaleConfig) -> RssImage:
    """Prescale -> per-coil forward 2-D FFT -> exact undo -> RSS (mri.py:84-91)."""
    if kspace.domain != KSPACE:
        raise InvalidValue("forward_pipeline expects a k-space grid")
    return _run_grid(kspace, plan, cfg, roundtrip=False)


def roundtrip_pipeline(image: ComplexGrid, plan: FftPlan, cfg: PrescaleConfig) -> RssImage:
    """Prescale -> per-coil forward then inverse 2-D FFT x 1/N^2 -> undo -> RSS
    (mri.py:94-107)."""
    if image.domain != IMAGE:
        raise InvalidValue("roundtrip_pipeline expects an image grid")
    return _run_grid(image, plan, cfg, roundtrip=True)
