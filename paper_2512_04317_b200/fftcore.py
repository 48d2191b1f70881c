"""Radix-2 DIT transforms with MX-scaled butterflies, on the GPU.

Public surface of pkg/src/mxfft/fftcore.py:32-353 (ModeSpec, FftPlan,
make_plan, butterfly_mx, fft_1d, fft_1d_fp16, fft_2d, plus the private
_fft_batch / _encode_blocks_batch / _mx_multiply_batch the reference tests
import).  Every ModeSpec kind runs in hand-written sm_100a kernels: MX behind
mxfft_fft_rows / mxfft_fft2 (csrc/mxfft_lines.cuh, csrc/mxfft_fft.cu), fp16
and reference behind mxfft_fft_rows_fp16 / mxfft_fft_rows_f64
(csrc/mxfft_modes.cu).  This module validates arguments, builds plans and
moves data.

The device-resident batched entry points (fft2_device, fft_rows_device) take
and return CUDA tensors without synchronizing; the numpy-facing functions are
thin wrappers over them.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np

from . import _native, mxblock
from .errors import InvalidValue, ShapeError, UnsupportedSize
from .minifloat import MinifloatFormat, get_format

MODE_CODES = {"forward": 0, "inverse": 1, "roundtrip": 2}


@dataclasses.dataclass(frozen=True)
class ModeSpec:
    """Arithmetic of a plan: "mx" (element format + block size B in reals),
    "fp16" (positive control) or "reference" (FP64)."""

    kind: str
    fmt: MinifloatFormat = None
    block_size: int = 32

    @staticmethod
    def mx(fmt: MinifloatFormat, block_size: int = 32) -> "ModeSpec":
        if block_size < 2 or block_size % 2 != 0:
            raise ValueError("block_size must be an even integer >= 2")
        return ModeSpec("mx", fmt, block_size)

    @staticmethod
    def fp16() -> "ModeSpec":
        return ModeSpec("fp16")

    @staticmethod
    def reference() -> "ModeSpec":
        return ModeSpec("reference")

    @staticmethod
    def from_name(name: str, block_size: int = 32) -> "ModeSpec":
        if name in ("reference", "fp16"):
            return ModeSpec(name)
        return ModeSpec.mx(get_format(name), block_size)

    @property
    def label(self) -> str:
        return self.fmt.name if self.kind == "mx" else self.kind


def _bit_reversal(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


def _twiddle_table(n: int) -> list:
    """FP64 twiddles per stage in butterfly order -- the reference's exact NumPy
    expression (fftcore.py:101-105), so the encoded plan matches bit-for-bit."""
    out = []
    stages = n.bit_length() - 1
    for s in range(stages):
        half = 1 << s
        step = n // (2 * half)
        w = np.exp(-2j * np.pi * np.arange(half) * step / n)
        out.append(np.tile(w, n // (2 * half)))
    return out


class FftPlan:
    """Per-size tables.  For "mx" plans the twiddles are encoded ONCE on the
    device (mxfft_plan_create) in the data's own format; the handle is
    read-only afterwards and safe to share across threads/streams."""

    def __init__(self, n: int, mode: ModeSpec):
        if n < 2 or n & (n - 1):
            raise UnsupportedSize(f"transform length must be a power of two >= 2, got {n}")
        self.n = n
        self.mode = mode
        self.stages = n.bit_length() - 1
        self.bitrev = _bit_reversal(n)
        self.ref_twiddles = _twiddle_table(n)
        self._handle = None
        self._mx_twiddles = None
        if mode.kind == "mx":
            self.cplx_per_block = min(mode.block_size // 2, n // 2)
            if (n // 2) % self.cplx_per_block:
                raise ValueError("block_size/2 must divide n/2")
            L = _native.lib()
            tw = np.ascontiguousarray(np.stack(self.ref_twiddles))
            h = ctypes.c_void_p()
            c = mode.fmt.as_c()
            _native.check(L.mxfft_plan_create(ctypes.byref(h), n, ctypes.byref(c),
                                              mode.block_size, tw.ctypes.data,
                                              _native.stream_handle()))
            self._handle = h
        elif mode.kind == "fp16":
            self.fp16_twiddles = [(w.real.astype(np.float16), w.imag.astype(np.float16))
                                  for w in self.ref_twiddles]

    def device_twiddles(self):
        """fp16 / reference plans: the n-entry device table (entry 2^s + j =
        twiddle j of stage s) the non-MX kernels read; built once from the
        plan's FP64 table (fp16: rounded by numpy exactly as the reference's
        plan, fftcore.py:115-117)."""
        import torch

        if getattr(self, "_dev_tw", None) is None:
            n = self.n
            if self.mode.kind == "fp16":
                t = np.zeros((n, 2), dtype=np.float16)
                for s, (wr, wi) in enumerate(self.fp16_twiddles):
                    half = 1 << s
                    t[half:2 * half, 0] = wr[:half]
                    t[half:2 * half, 1] = wi[:half]
                self._dev_tw = torch.from_numpy(t.view(np.uint8).reshape(-1).copy()).cuda()
            elif self.mode.kind == "reference":
                t = np.zeros(n, dtype=np.complex128)
                for s, w in enumerate(self.ref_twiddles):
                    half = 1 << s
                    t[half:2 * half] = w[:half]
                self._dev_tw = torch.from_numpy(t).cuda()
            else:
                raise ValueError("MX plans keep their tables behind the plan handle")
        return self._dev_tw

    @property
    def handle(self):
        if self._handle is None:
            raise ValueError("plan has no device tables (mode is not 'mx')")
        return self._handle

    @property
    def mx_twiddles(self):
        """[(codes_re (1, nb, cpb), codes_im, scales (1, nb))] per stage, read
        back from the device tables (fftcore.py:110-113 layout)."""
        if self._mx_twiddles is None:
            m, cpb = self.n // 2, self.cplx_per_block
            nb = m // cpb
            cr = np.empty((self.stages, m))
            ci = np.empty((self.stages, m))
            sc = np.empty((self.stages, nb))
            _native.check(_native.lib().mxfft_plan_twiddles(self.handle, cr.ctypes.data,
                                                            ci.ctypes.data, sc.ctypes.data))
            self._mx_twiddles = [(cr[s].reshape(1, nb, cpb), ci[s].reshape(1, nb, cpb),
                                  sc[s].reshape(1, nb)) for s in range(self.stages)]
        return self._mx_twiddles

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and _native._lib is not None:
            try:
                _native._lib.mxfft_plan_destroy(h)
            except Exception:
                pass


def make_plan(n: int, mode: ModeSpec) -> FftPlan:
    return FftPlan(n, mode)


_HW_FORMATS = {("e4m3", 4, 3, "extended", 7), ("e5m2", 5, 2, "ieee", 15),
               ("e2m3", 2, 3, "finite", 1), ("e3m2", 3, 2, "finite", 3),
               ("e2m1", 2, 1, "finite", 1)}


def fast_path_supported(plan: FftPlan) -> bool:
    """True when the plan runs on the register/shared-memory line kernel with
    hardware quantizers (mirrors fast_path_ok in csrc/mxfft_fft.cu); other plans
    use the generic reference-literal kernel."""
    if plan.mode.kind != "mx":
        return False
    f = plan.mode.fmt
    ids = {(a, b, c, d) for (_, a, b, c, d) in _HW_FORMATS}
    if (f.exponent_bits, f.mantissa_bits, f.policy, f.bias) not in ids:
        return False
    cpb = plan.cplx_per_block
    if cpb > 32 or cpb & (cpb - 1):
        return False
    logch = 6 if 2 * cpb > 32 else 5
    if plan.stages < logch:
        return False
    return (plan.n >> logch) <= (256 if logch == 6 else 512)


# ---------------------------------------------------------------------------
# device-resident batched API
# ---------------------------------------------------------------------------
def _require_mx(plan: FftPlan):
    if plan.mode.kind != "mx":
        raise NotImplementedError(
            f"the batched device entry points take MX plans; {plan.mode.kind!r} plans run through "
            "_fft_batch / fft_1d / fft_2d (mxfft_fft_rows_fp16 / mxfft_fft_rows_f64)")


def fft_rows_device(x, plan: FftPlan, inverse: bool = False, out=None):
    """Batched 1-D MX transform of the rows of a CUDA complex64 tensor (..., n)."""
    import torch

    _require_mx(plan)
    if x.dtype != torch.complex64 or not x.is_cuda:
        raise TypeError("expected a CUDA complex64 tensor")
    if x.shape[-1] != plan.n:
        raise ShapeError(f"expected length {plan.n}, got {x.shape[-1]}")
    x = x.contiguous()
    y = out if out is not None else torch.empty_like(x)
    rows = x.numel() // plan.n
    _native.check(_native.lib().mxfft_fft_rows(plan.handle, x.data_ptr(), y.data_ptr(), rows,
                                               int(bool(inverse)), _native.stream_handle()))
    return y


def fft_cols_device(x, plan: FftPlan, inverse: bool = False, out=None):
    """Batched 1-D MX transform along the columns of CUDA complex64 images (B, n, n)."""
    import torch

    _require_mx(plan)
    if x.dtype != torch.complex64 or not x.is_cuda or x.shape[-1] != plan.n \
            or x.shape[-2] != plan.n:
        raise ShapeError("expected CUDA complex64 images (B, n, n)")
    x = x.contiguous()
    y = out if out is not None else torch.empty_like(x)
    batch = x.numel() // (plan.n * plan.n)
    _native.check(_native.lib().mxfft_fft_cols(plan.handle, x.data_ptr(), y.data_ptr(), batch,
                                               int(bool(inverse)), _native.stream_handle()))
    return y


def fft2_device(x, plan: FftPlan, mode: str = "forward", k=None, k_group: int = 1, out=None,
                workspace=None):
    """Batched 2-D MX transform of CUDA complex64 images (B, n, n).

    mode: "forward" | "inverse" | "roundtrip" (forward, inverse, x 1/n^2).
    k: optional CUDA int32 tensor of prescale exponents, one per k_group
    images; fuses apply_prescale on load and undo_prescale on store.
    workspace: None = take a scratch buffer from torch's caching allocator
    (every pass is then a row pass with a transposed store); a CUDA tensor of
    at least mxfft_fft2_workspace_bytes bytes; or False = no scratch (the
    column pass runs in place on the output, same results)."""
    import torch

    _require_mx(plan)
    if x.dtype != torch.complex64 or not x.is_cuda:
        raise TypeError("expected a CUDA complex64 tensor")
    if x.dim() < 2 or x.shape[-1] != x.shape[-2]:
        raise UnsupportedSize("fft_2d expects square grids")
    if x.shape[-1] != plan.n:
        raise UnsupportedSize(f"grid size {x.shape[-1]} does not match plan size {plan.n}")
    x = x.contiguous()
    y = out if out is not None else torch.empty_like(x)
    batch = x.numel() // (plan.n * plan.n)
    kp = None
    if k is not None:
        if k.dtype != torch.int32 or not k.is_cuda:
            raise TypeError("k must be a CUDA int32 tensor")
        if k_group < 1 or k.numel() * k_group < batch:
            raise ShapeError(f"{k.numel()} prescale exponents x k_group {k_group} do not cover {batch} images")
        kp = k.data_ptr()
    L = _native.lib()
    wp, wb = None, 0
    if workspace is not False:
        need = int(L.mxfft_fft2_workspace_bytes(plan.handle, batch))
        if need > 0:
            if workspace is None:
                workspace = torch.empty(need, dtype=torch.uint8, device=x.device)
            wp, wb = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    _native.check(L.mxfft_fft2(plan.handle, x.data_ptr(), y.data_ptr(), batch, MODE_CODES[mode],
                               kp, int(k_group), wp, wb, _native.stream_handle()))
    return y


def fft_rows_debug(x, plan: FftPlan, inverse: bool = False):
    """Per-stage capture of the row transform (test instrumentation): returns
    (y, dict(v_exp, v_codes, p_exp, p_shift, p_codes, stage_out)) as numpy."""
    import torch

    _require_mx(plan)
    x = x.contiguous()
    rows = x.numel() // plan.n
    st, m, cpb = plan.stages, plan.n // 2, plan.cplx_per_block
    nb = m // cpb
    dev = x.device
    cap = dict(
        v_exp=torch.empty((st, rows, nb), dtype=torch.int32, device=dev),
        v_codes=torch.empty((st, rows, m, 2), dtype=torch.float32, device=dev),
        p_exp=torch.empty((st, rows, nb), dtype=torch.int32, device=dev),
        p_shift=torch.empty((st, rows, nb), dtype=torch.int32, device=dev),
        p_codes=torch.empty((st, rows, m, 2), dtype=torch.float32, device=dev),
        stage_out=torch.empty((st, rows, plan.n), dtype=torch.complex64, device=dev),
    )
    y = torch.empty_like(x)
    _native.check(_native.lib().mxfft_fft_rows_debug(
        plan.handle, x.data_ptr(), y.data_ptr(), rows, int(bool(inverse)),
        cap["v_exp"].data_ptr(), cap["v_codes"].data_ptr(), cap["p_exp"].data_ptr(),
        cap["p_shift"].data_ptr(), cap["p_codes"].data_ptr(), cap["stage_out"].data_ptr(),
        _native.stream_handle()))
    return y.cpu().numpy(), {k: v.cpu().numpy() for k, v in cap.items()}


# ---------------------------------------------------------------------------
# numpy-facing reference API
# ---------------------------------------------------------------------------
def _to_c64_device(x: np.ndarray):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).cuda().to(torch.complex64)


def _fft_batch(x: np.ndarray, plan: FftPlan, direction: str) -> np.ndarray:
    if direction not in ("forward", "inverse"):
        raise ValueError(f"direction must be 'forward' or 'inverse', got {direction!r}")
    x = np.asarray(x)
    if x.shape[1] != plan.n:
        raise ShapeError(f"expected length {plan.n}, got {x.shape[1]}")
    inverse = direction == "inverse"
    if plan.mode.kind == "fp16":
        return _fft_rows_fp16(x, plan, inverse)
    if plan.mode.kind == "reference":
        return _fft_rows_f64(x, plan, inverse)
    y = fft_rows_device(_to_c64_device(x), plan, inverse)
    return y.cpu().numpy()


def _fft_rows_fp16(x: np.ndarray, plan: FftPlan, inverse: bool) -> np.ndarray:
    """_fft_batch_fp16 (fftcore.py:285-311) on the GPU: complex64 input is
    quantized from FP32, anything else from FP64, as the reference does."""
    import torch

    c64 = x.dtype == np.complex64
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex64 if c64 else np.complex128)).cuda()
    y = torch.empty(xd.shape, dtype=torch.complex64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _native.check(_native.lib().mxfft_fft_rows_fp16(xd.data_ptr(), int(not c64), y.data_ptr(), xd.shape[0],
                                                    plan.n, plan.device_twiddles().data_ptr(), int(inverse),
                                                    flag.data_ptr(), _native.stream_handle()))
    if int(flag.item()):
        raise InvalidValue("non-finite value in the FP16 transform (quantize_array)")
    return y.cpu().numpy()


def _fft_rows_f64(x: np.ndarray, plan: FftPlan, inverse: bool) -> np.ndarray:
    """_fft_batch_reference (fftcore.py:243-256) on the GPU, complex128."""
    import torch

    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).cuda()
    y = torch.empty_like(xd)
    _native.check(_native.lib().mxfft_fft_rows_f64(xd.data_ptr(), y.data_ptr(), xd.shape[0], plan.n,
                                                   plan.device_twiddles().data_ptr(), int(inverse),
                                                   _native.stream_handle()))
    return y.cpu().numpy()


def fft_1d(x, plan: FftPlan, direction: str = "forward") -> np.ndarray:
    """Unnormalized radix-2 DIT transform of one length-n vector."""
    x = np.asarray(x, dtype=np.complex128)
    if x.ndim != 1:
        raise ShapeError("fft_1d expects a 1-D vector")
    return _fft_batch(x[None, :], plan, direction)[0]


def fft_1d_fp16(x, plan: FftPlan, direction: str = "forward") -> np.ndarray:
    if plan.mode.kind != "fp16":
        raise ValueError("fft_1d_fp16 requires an fp16-mode plan")
    return fft_1d(x, plan, direction)


def fft_2d(x, plan: FftPlan, direction: str = "forward") -> np.ndarray:
    """Rows, then columns, of a square n x n grid (fftcore.py:344-353)."""
    x = np.asarray(x, dtype=np.complex128)
    if x.ndim != 2 or x.shape[0] != x.shape[1]:
        raise UnsupportedSize("fft_2d expects a square grid")
    if x.shape[0] != plan.n:
        raise UnsupportedSize(f"grid size {x.shape[0]} does not match plan size {plan.n}")
    if direction not in ("forward", "inverse"):
        raise ValueError(f"direction must be 'forward' or 'inverse', got {direction!r}")
    if plan.mode.kind != "mx":  # fp16 / reference: rows, rows.T, cols.T as fftcore.py:351-353
        rows = _fft_batch(x, plan, direction)
        cols = _fft_batch(np.ascontiguousarray(rows.T), plan, direction)
        return np.asarray(cols.T, dtype=np.complex128)
    y = fft2_device(_to_c64_device(x[None]), plan, direction)
    return y[0].cpu().numpy().astype(np.complex128)


def _encode_blocks_batch(vr, vi, cpb: int, fmt: MinifloatFormat):
    """(batch, m) real/imag -> codes_r, codes_i (batch, nb, cpb), scales (batch, nb);
    one scale per cpb complex values (fftcore.py:131-147), encoded on the GPU."""
    vr = np.asarray(vr, dtype=np.float64)
    vi = np.asarray(vi, dtype=np.float64)
    b, m = vr.shape
    nb = m // cpb
    inter = np.empty((b, nb, 2 * cpb))
    inter[..., 0::2] = vr.reshape(b, nb, cpb)
    inter[..., 1::2] = vi.reshape(b, nb, cpb)
    codes, scales = mxblock._encode_rows(inter.reshape(b * nb, 2 * cpb), fmt)
    codes = codes.reshape(b, nb, 2 * cpb)
    return codes[..., 0::2].copy(), codes[..., 1::2].copy(), scales.reshape(b, nb)


def _mx_multiply_kernel(vr, vi, w_enc, fmt: MinifloatFormat, cpb: int, u=None):
    """mxfft_mx_multiply_f64: the blockwise MX complex product w*v of
    fftcore.py:150-183 (and, given u, the butterfly of fftcore.py:186-235) in
    one CUDA kernel.  Returns wv complex128 (batch, m) [, y0, y1 complex64]."""
    import torch

    vr = np.asarray(vr, dtype=np.float64)
    vi = np.asarray(vi, dtype=np.float64)
    b, m = vr.shape
    wcr, wci, ws = (np.ascontiguousarray(np.asarray(t, dtype=np.float64)) for t in w_enc)
    nb = m // cpb
    if wcr.size != nb * cpb or ws.size != nb:
        raise ShapeError("twiddle blocks do not match the operand length")
    v = torch.from_numpy(np.ascontiguousarray(vr + 1j * vi)).cuda()
    dev = [torch.from_numpy(t.reshape(-1)).cuda() for t in (wcr, wci, ws)]
    wv = torch.empty((b, m), dtype=torch.complex128, device="cuda")
    nf = torch.zeros(1, dtype=torch.int32, device="cuda")
    args = [None, None, None]
    if u is not None:
        ud = torch.from_numpy(np.ascontiguousarray(np.asarray(u, dtype=np.complex128).reshape(b, m))).cuda()
        y0 = torch.empty((b, m), dtype=torch.complex64, device="cuda")
        y1 = torch.empty_like(y0)
        args = [ud.data_ptr(), y0.data_ptr(), y1.data_ptr()]
    c = fmt.as_c()
    _native.check(_native.lib().mxfft_mx_multiply_f64(v.data_ptr(), dev[0].data_ptr(), dev[1].data_ptr(),
                                                      dev[2].data_ptr(), b, m, cpb, ctypes.byref(c), wv.data_ptr(),
                                                      *args, nf.data_ptr(), _native.stream_handle()))
    if int(nf.item()):
        raise InvalidValue("non-finite block element")
    if u is not None:
        return wv.cpu().numpy(), y0.cpu().numpy(), y1.cpu().numpy()
    return wv.cpu().numpy()


def _mx_multiply_batch(vr, vi, w_enc, fmt: MinifloatFormat, cpb: int) -> np.ndarray:
    """Blockwise MX complex multiply w*v for a whole stage (fftcore.py:150-183),
    on the GPU (mxfft_mx_multiply_f64)."""
    return _mx_multiply_kernel(vr, vi, w_enc, fmt, cpb)


def butterfly_mx(u, v, w, fmt: MinifloatFormat):
    """One MX-scaled complex butterfly on a block of up to B/2 values (literal
    single-block procedure, fftcore.py:186-235); returns (u + wv, u - wv) in FP32."""
    u = np.asarray(u, dtype=np.complex128)
    v = np.asarray(v, dtype=np.complex128)
    if isinstance(w, mxblock.MxBlock):
        w_blk = w
    else:
        w = np.asarray(w, dtype=np.complex128)
        inter = np.empty(2 * w.size)
        inter[0::2], inter[1::2] = w.real, w.imag
        w_blk = mxblock.encode_block_mx(inter, fmt)
    if u.shape != v.shape or 2 * v.size != w_blk.n:
        raise ShapeError("butterfly operands must have matching lengths")
    cpb = v.size
    wr, wi = mxblock.mantissas_block(w_blk)
    w_enc = (wr.reshape(1, cpb), wi.reshape(1, cpb), np.array([w_blk.scale]))
    _, y0, y1 = _mx_multiply_kernel(v.real[None], v.imag[None], w_enc, fmt, cpb, u=u[None])
    return y0[0], y1[0]
