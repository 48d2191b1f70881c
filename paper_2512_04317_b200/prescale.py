"""Global power-of-two prescale (Alg. 1 of the paper) and its exact inverse.

Same API as pkg/src/mxfft/prescale.py:21-91.  The statistics (peak magnitude,
tau-percentile of the nonzero magnitudes, k) are computed on the GPU by
mxfft_prescale_stats: a fused amax + histogram radix-select kernel.  The one
scalar decision the host keeps is re-deriving k when the device flags a log2
that landed within a few ulps of a rounding boundary (never for real data).
"""

from __future__ import annotations

import ctypes
import dataclasses
import math

import numpy as np

from . import _native
from .errors import ConfigError, InvalidValue

EPS = 1e-30  # log2 guard for an all-zero peak or tail (prescale.py:18)


@dataclasses.dataclass(frozen=True)
class PrescaleConfig:
    target: float = 1.0
    tau: float = 1.0  # percentile (in percent) of the nonzero magnitudes
    tau_min: float = 2.0**-20
    k_min: int = -40
    k_max: int = 40

    def __post_init__(self):
        if not self.target > 0:
            raise ConfigError("target", "must be > 0")
        if not 0 < self.tau < 100:
            raise ConfigError("tau", "must be in (0, 100)")
        if not self.tau_min > 0:
            raise ConfigError("tau_min", "must be > 0")
        if self.k_min > self.k_max:
            raise ConfigError("k_min", "must be <= k_max")

    def as_c(self) -> _native.PrescaleCfgC:
        return _native.PrescaleCfgC(float(self.target), float(self.tau), float(self.tau_min),
                                    int(self.k_min), int(self.k_max))


@dataclasses.dataclass(frozen=True)
class PrescaleResult:
    k: int
    a_max: float
    p_tau: float
    k1: int
    k2: int


def k_from_stats(a_max: float, p_tau: float, cfg: PrescaleConfig):
    """The scalar k rule (prescale.py:70-72) evaluated with the host's log2."""
    v = math.log2(cfg.target / max(a_max, EPS))
    k1 = math.floor(v + 0.5) if v >= 0 else math.ceil(v - 0.5)
    k2 = math.ceil(math.log2(cfg.tau_min / max(p_tau, EPS)))
    return min(max(max(k1, k2), cfg.k_min), cfg.k_max), k1, k2


_WS = {}  # (device, stream, nbytes) -> reusable workspace of the sampled statistics path


def _workspace(device, nbytes: int):
    """Scratch of the statistics kernels, one per (device, stream, size): work
    on different streams (or a captured graph replaying beside eager calls on
    another stream) never shares it."""
    import torch

    if nbytes <= 0:
        return None
    key = (str(device), _native.stream_handle(), nbytes)
    if key not in _WS:
        _WS[key] = torch.empty(nbytes, dtype=torch.uint8, device=device)
    return _WS[key]


def prescale_stats_device(x, nseg: int, seg_points: int, cfg: PrescaleConfig, k_out=None,
                          res_out=None, workspace=None):
    """Launch the statistics kernels on a CUDA tensor (complex64 or complex128,
    nseg contiguous segments of seg_points values) without synchronizing.
    Returns (results uint8 tensor (nseg, 40), k int32 tensor (nseg,)).

    complex64 segments use the sampled fast path (needs a device workspace of
    mxfft_prescale_workspace_bytes; one is cached per size when not given);
    complex128 and unsettled segments use the exact histogram kernel."""
    import torch

    L = _native.lib()
    if x.dtype not in (torch.complex64, torch.complex128):
        raise TypeError("prescale statistics take complex64 or complex128 data")
    res = res_out if res_out is not None else torch.empty(
        (nseg, _native.PRESCALE_RESULT_DTYPE.itemsize), dtype=torch.uint8, device=x.device)
    k = k_out if k_out is not None else torch.empty(nseg, dtype=torch.int32, device=x.device)
    c = cfg.as_c()
    ws_ptr, ws_bytes = None, 0
    if x.dtype == torch.complex64:
        need = int(L.mxfft_prescale_workspace_bytes(nseg, seg_points))
        ws = workspace if workspace is not None and workspace.numel() >= need else \
            _workspace(x.device, need)
        if ws is not None:
            ws_ptr, ws_bytes = ws.data_ptr(), ws.numel()
    _native.check(L.mxfft_prescale_stats(x.data_ptr(), int(x.dtype == torch.complex128), nseg,
                                         seg_points, ctypes.byref(c), res.data_ptr(), k.data_ptr(),
                                         ws_ptr, ws_bytes, _native.stream_handle()))
    return res, k


def decode_results(res) -> np.ndarray:
    """Device result rows -> numpy structured array (a_max, p_tau, k1, k2, k, flags, nnz)."""
    return np.frombuffer(res.cpu().numpy().tobytes(), dtype=_native.PRESCALE_RESULT_DTYPE)


def _is_grid(x) -> bool:
    return not isinstance(x, np.ndarray) and hasattr(x, "data")


def _data_of(x) -> np.ndarray:
    return np.asarray(x.data if _is_grid(x) else x)


def compute_prescale(x, cfg: PrescaleConfig) -> PrescaleResult:
    """Choose k for input x (array or grid) over all of its values."""
    import torch

    data = np.asarray(_data_of(x))
    c = np.ascontiguousarray(data, dtype=np.complex128).reshape(-1)
    if c.size == 0:
        raise ValueError("zero-size array")
    t = torch.from_numpy(c).cuda()
    res, _ = prescale_stats_device(t, 1, c.size, cfg)
    r = decode_results(res)[0]
    if int(r["flags"]) & 1:
        raise InvalidValue("non-finite input to prescale")
    a_max, p_tau = float(r["a_max"]), float(r["p_tau"])
    k, k1, k2 = int(r["k"]), int(r["k1"]), int(r["k2"])
    if int(r["flags"]) & 2:
        k, k1, k2 = k_from_stats(a_max, p_tau, cfg)
    return PrescaleResult(k=k, a_max=a_max, p_tau=p_tau, k1=k1, k2=k2)


def _scale_array(arr: np.ndarray, k: int) -> np.ndarray:
    """arr * math.ldexp(1.0, k) with numpy's dtype rules (prescale.py:83),
    computed by the mxfft_scale kernel:
    - float32 / complex64 stay single precision, with the factor rounded to
      float32 first (numpy rounds the weak Python float the same way);
    - float64 / complex128 stay double;
    - float16 is multiplied in single precision and rounded back once (what
      numpy's float16 multiply does), with the factor rounded to float16;
    - everything else (ints, bools) is promoted to float64."""
    import torch

    f64 = math.ldexp(1.0, k)  # OverflowError for k >= 1024, as in the reference
    with np.errstate(over="ignore"):
        if arr.dtype in (np.float32, np.complex64):
            work, factor, is_f64, back = arr, float(np.float32(f64)), 0, None
        elif arr.dtype in (np.float64, np.complex128):
            work, factor, is_f64, back = arr, f64, 1, None
        elif arr.dtype == np.float16:
            work, factor, is_f64, back = arr.astype(np.float32), float(np.float16(f64)), 0, np.float16
        else:
            work, factor, is_f64, back = arr.astype(np.float64), f64, 1, None
    flat = np.ascontiguousarray(work).reshape(-1)
    cplx = flat.dtype.kind == "c"
    real = flat.view(np.float64 if is_f64 else np.float32) if cplx else flat
    t = torch.from_numpy(real).cuda()
    out = torch.empty_like(t)
    _native.check(_native.lib().mxfft_scale(t.data_ptr(), out.data_ptr(), flat.size, is_f64 + 2 * cplx, factor,
                                           _native.stream_handle()))
    res = out.cpu().numpy().view(flat.dtype).reshape(arr.shape)
    return res.astype(back) if back is not None else res


def apply_prescale(x, k: int):
    """x * 2^k (prescale.py:76-86), on the GPU; returns the same kind of object
    (array or grid)."""
    data = _data_of(x)
    scaled = _scale_array(np.asarray(data), int(k))
    if _is_grid(x):
        return dataclasses.replace(x, data=scaled)
    return scaled


def undo_prescale(x, k: int):
    """Exact inverse of apply_prescale (prescale.py:89-91)."""
    return apply_prescale(x, -k)
