"""MX block codec: B real scalars sharing one power-of-two scale.

Public surface of pkg/src/mxfft/mxblock.py:19-90; the arithmetic runs on the
GPU (mxfft_mx_encode_f64 / mxfft_mx_decode_f64 / mxfft_quantize_f64).
Complex values are interleaved (re, im), so a block of B reals carries B/2
complex values under one scale; codes are the decoded element-format reals.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _native
from .errors import InvalidValue, MantissaOverflow, ShapeError
from .minifloat import MinifloatFormat, quantize_array


@dataclasses.dataclass(frozen=True)
class MxBlock:
    codes: np.ndarray  # element-format reals, length n
    scale: float  # exact power of two
    n: int
    fmt: MinifloatFormat


def _encode_rows(rows: np.ndarray, fmt: MinifloatFormat):
    """Encode each row of a (nblocks, len) FP64 array as one MX block on the GPU.
    Returns (codes (nblocks, len), scales (nblocks,))."""
    import torch

    L = _native.lib()
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    nb, ln = rows.shape
    t = torch.from_numpy(rows).cuda()
    codes = torch.empty_like(t)
    scales = torch.empty(nb, dtype=torch.float64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    c = fmt.as_c()
    _native.check(L.mxfft_mx_encode_f64(t.data_ptr(), nb, ln, ctypes.byref(c), codes.data_ptr(),
                                        scales.data_ptr(), flag.data_ptr(),
                                        _native.stream_handle()))
    if int(flag.item()):
        raise InvalidValue("non-finite block element")
    return codes.cpu().numpy(), scales.cpu().numpy()


def block_scales(amax, fmt: MinifloatFormat) -> np.ndarray:
    """2^(floor(log2 amax) - emax) per value, 1.0 where amax == 0
    (mxblock.py:27-38): the scale the encoder picks for a block whose largest
    magnitude is amax."""
    a = np.asarray(amax, dtype=np.float64)
    if a.size == 0:
        return np.ones(a.shape)
    _, s = _encode_rows(np.abs(a).reshape(-1, 1), fmt)
    return s.reshape(a.shape)


def encode_block_mx(values, fmt: MinifloatFormat) -> MxBlock:
    v = np.asarray(values, dtype=np.float64)
    if v.ndim != 1 or v.size < 1:
        raise ShapeError("block must be a non-empty 1-D array")
    if not np.all(np.isfinite(v)):
        raise InvalidValue("non-finite block element")
    codes, scales = _encode_rows(v[None, :], fmt)
    return MxBlock(codes[0], float(scales[0]), v.size, fmt)


def mantissas_block(b: MxBlock):
    """(real codes, imag codes) of a block, scale not applied."""
    if b.n % 2:
        raise ShapeError("complex block length must be even")
    return b.codes[0::2].copy(), b.codes[1::2].copy()


def encode_from_mant_block(p_r, p_i, s_out: float, fmt: MinifloatFormat) -> MxBlock:
    """Quantize already-renormalized mantissa-space values as a block with scale
    s_out; raises MantissaOverflow if a value exceeds max_finite (a missed
    renormalization)."""
    p_r = np.asarray(p_r, dtype=np.float64)
    p_i = np.asarray(p_i, dtype=np.float64)
    if p_r.ndim != 1 or p_r.shape != p_i.shape:
        raise ShapeError("mantissa vectors must be 1-D and of equal length")
    inter = np.empty(2 * p_r.size, dtype=np.float64)
    inter[0::2] = p_r
    inter[1::2] = p_i
    amax = float(np.max(np.abs(inter), initial=0.0))
    if amax > fmt.max_finite:
        raise MantissaOverflow(f"mantissa magnitude {amax} exceeds {fmt.name} max {fmt.max_finite}")
    codes = quantize_array(inter, fmt)
    return MxBlock(codes, float(s_out), codes.size, fmt)


def decode_block_mx(b: MxBlock) -> np.ndarray:
    """The B/2 complex values codes * scale, FP64 (on the GPU)."""
    import torch

    if b.n % 2:
        raise ShapeError("complex block length must be even")
    L = _native.lib()
    codes = torch.from_numpy(np.ascontiguousarray(b.codes, dtype=np.float64)).cuda()
    scales = torch.tensor([float(b.scale)], dtype=torch.float64, device="cuda")
    out = torch.empty(b.n, dtype=torch.float64, device="cuda")
    _native.check(L.mxfft_mx_decode_f64(codes.data_ptr(), scales.data_ptr(), 1, b.n,
                                        out.data_ptr(), _native.stream_handle()))
    return out.cpu().numpy().view(np.complex128)
