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

import dataclasses

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
def pipeline_device(x, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool, coils: int = 1,
                    out=None, k=None, res=None):
    """x: CUDA complex64 (B*coils, N, N).  Stacks of `coils` consecutive images
    share one prescale (C = 1: per image).  Returns (out complex64, k int32 (B,),
    stats uint8 (B, 40)) without synchronizing."""
    n = plan.n
    nstack = x.shape[0] // coils
    res, k = prescale_stats_device(x, nstack, coils * n * n, cfg, k_out=k, res_out=res)
    y = fft2_device(x, plan, "roundtrip" if roundtrip else "forward", k=k, k_group=coils, out=out)
    return y, k, res


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
                  coils: int = 1, chunks: int = 8, graph: bool = True):
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
           repr(cfg), bool(roundtrip), int(coils), int(chunks))
    ent = _HOST_GRAPHS.get(key)
    if ent is None or ent[1] is not plan:
        _pipeline_host_eager(x_host, plan, cfg, roundtrip, out_host, coils, chunks)  # warm-up
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cs):
            _pipeline_host_eager(x_host, plan, cfg, roundtrip, out_host, coils, chunks, capture=True)
        if len(_HOST_GRAPHS) >= _HOST_GRAPHS_MAX:
            _HOST_GRAPHS.pop(next(iter(_HOST_GRAPHS)))
        ent = (g, plan)
        _HOST_GRAPHS[key] = ent
    ent[0].replay()
    torch.cuda.current_stream().synchronize()
    return out_host


def _pipeline_host_eager(x_host, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool, out_host=None,
                         coils: int = 1, chunks: int = 8, capture: bool = False):
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
    nstack = x_host.shape[0] // coils
    if out_host is None:
        out_host = torch.empty(x_host.shape, dtype=x_host.dtype).pin_memory()
    if nstack == 0:
        return out_host
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
            pipeline_device(xs, plan, cfg, roundtrip, coils=coils, out=ys, k=ks)
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
    return out_host


def _run_grid(grid: ComplexGrid, plan: FftPlan, cfg: PrescaleConfig, roundtrip: bool) -> RssImage:
    import torch

    x128 = torch.from_numpy(np.ascontiguousarray(grid.data)).cuda()
    # statistics on the caller's FP64 values (prescale.py:66-69), transform in complex64
    res, k = prescale_stats_device(x128, 1, x128.numel(), cfg)
    x = x128.to(torch.complex64)
    y = fft2_device(x, plan, "roundtrip" if roundtrip else "forward", k=k, k_group=grid.coils)
    r = decode_results(res)[0]
    if int(r["flags"]) & 1:
        raise InvalidValue("non-finite input to prescale")
    if int(r["flags"]) & 2:  # k near a log2 rounding boundary: decide on the host
        kh, _, _ = k_from_stats(float(r["a_max"]), float(r["p_tau"]), cfg)
        if kh != int(r["k"]):
            k = torch.tensor([kh], dtype=torch.int32, device=x.device)
            y = fft2_device(x, plan, "roundtrip" if roundtrip else "forward", k=k,
                            k_group=grid.coils)
    return RssImage(rss_device(y, coils=grid.coils)[0].cpu().numpy())


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
