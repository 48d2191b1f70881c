"""ctypes front-end of the CPU oracle (oracle/mxfft_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs, never by the product package.  It is the checker
the CUDA path is compared against.  Each wrapper names the reference function
(/root/reference/pkg/src/mxfft/...) whose semantics the C code restates.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

POLICY_CODES = {"ieee": 0, "extended": 1, "finite": 2}


def build() -> str:
    """Compile the oracle (make -C oracle); returns the .so path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "mxfft_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        ip = ctypes.POINTER(ctypes.c_int)
        i32p = ctypes.POINTER(ctypes.c_int32)
        c_long, c_int, c_double = ctypes.c_long, ctypes.c_int, ctypes.c_double
        fmt4 = [c_int, c_int, c_int, c_int]
        L.orc_format_info.argtypes = fmt4 + [ip, ip, dp, dp]
        L.orc_quantize_array.argtypes = [dp, dp, c_long] + fmt4
        L.orc_quantize_array.restype = c_int
        L.orc_block_scales.argtypes = [dp, dp, c_long] + fmt4
        L.orc_encode_blocks.argtypes = [dp, dp, c_long, c_long, c_int] + fmt4 + [dp, dp, dp]
        L.orc_encode_twiddles.argtypes = [dp, c_int, c_int] + fmt4 + [dp, dp, dp]
        L.orc_fft_batch_mx.argtypes = (
            [dp, c_long, c_int, c_int] + fmt4 + [dp, dp, dp, c_int, fp, ctypes.c_void_p]
        )
        L.orc_fft_batch_mx.restype = c_int
        L.orc_fft2_mx.argtypes = [dp, c_int, c_int] + fmt4 + [dp, dp, dp, c_int, fp]
        L.orc_fft2_mx.restype = c_int
        L.orc_compute_prescale.argtypes = [dp, c_long, c_int, c_double, c_double, c_double, c_int,
                                           c_int, dp, dp, ip, ip, ip]
        L.orc_compute_prescale.restype = c_int
        L.orc_pipeline.argtypes = ([dp, c_int, c_int, c_int] + fmt4 + [dp, dp, dp, c_double,
                                   c_double, c_double, c_int, c_int, c_int, dp, dp, ip])
        L.orc_pipeline.restype = c_int
        L.orc_cabs.argtypes = [dp, c_long, dp]
        _ = i32p
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


@dataclass(frozen=True)
class Fmt:
    """(1, E, M) element format, minifloat.py:28-85."""

    name: str
    ebits: int
    mbits: int
    policy: str = "finite"
    bias: int | None = None

    @property
    def resolved_bias(self) -> int:
        return (1 << (self.ebits - 1)) - 1 if self.bias is None else self.bias

    @property
    def args(self):
        return (self.ebits, self.mbits, POLICY_CODES[self.policy], self.resolved_bias)

    def info(self):
        emin, emax = ctypes.c_int(), ctypes.c_int()
        mf, ms = ctypes.c_double(), ctypes.c_double()
        lib().orc_format_info(*self.args, ctypes.byref(emin), ctypes.byref(emax),
                              ctypes.byref(mf), ctypes.byref(ms))
        return dict(emin=emin.value, emax=emax.value, max_finite=mf.value,
                    min_subnormal=ms.value)


E4M3 = Fmt("e4m3", 4, 3, "extended")
E5M2 = Fmt("e5m2", 5, 2, "ieee")
E2M3 = Fmt("e2m3", 2, 3, "finite")
E3M2 = Fmt("e3m2", 3, 2, "finite")
E2M1 = Fmt("e2m1", 2, 1, "finite")
FP16 = Fmt("fp16", 5, 10, "ieee")
WIDE = Fmt("wide", 8, 23, "ieee")
ALL_MX = {f.name: f for f in (E4M3, E5M2, E2M3, E3M2, E2M1)}


def as_fmt(f) -> Fmt:
    """Accept an oracle Fmt or any object with the reference's MinifloatFormat fields."""
    if isinstance(f, Fmt):
        return f
    return Fmt(f.name, f.exponent_bits, f.mantissa_bits, f.policy, f.bias)


def quantize_array(x, fmt) -> np.ndarray:
    """minifloat.py:105-120."""
    fmt = as_fmt(fmt)
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    out = np.empty_like(x)
    rc = lib().orc_quantize_array(_dp(x), _dp(out), x.size, *fmt.args)
    if rc:
        raise ValueError("non-finite input to quantize")
    return out


def block_scales(amax, fmt) -> np.ndarray:
    """mxblock.py:27-38."""
    fmt = as_fmt(fmt)
    a = np.ascontiguousarray(np.asarray(amax, dtype=np.float64))
    out = np.empty_like(a)
    lib().orc_block_scales(_dp(a), _dp(out), a.size, *fmt.args)
    return out


def encode_blocks(vr, vi, cpb, fmt):
    """_encode_blocks_batch, fftcore.py:131-147 -> (codes_r, codes_i, scales)."""
    fmt = as_fmt(fmt)
    vr = np.ascontiguousarray(np.asarray(vr, dtype=np.float64))
    vi = np.ascontiguousarray(np.asarray(vi, dtype=np.float64))
    b, m = vr.shape
    cr = np.empty((b, m))
    ci = np.empty((b, m))
    sc = np.empty((b, m // cpb))
    lib().orc_encode_blocks(_dp(vr), _dp(vi), b, m, cpb, *fmt.args, _dp(cr), _dp(ci), _dp(sc))
    return cr.reshape(b, m // cpb, cpb), ci.reshape(b, m // cpb, cpb), sc


def ref_twiddles(n: int) -> np.ndarray:
    """FP64 twiddles in butterfly order, (stages, n/2) -- the reference's own NumPy
    expression (fftcore.py:101-105), evaluated term by term in the same order."""
    stages = n.bit_length() - 1
    out = np.empty((stages, n // 2), dtype=np.complex128)
    for s in range(stages):
        half = 1 << s
        step = n // (2 * half)
        w = np.exp(-2j * np.pi * np.arange(half) * step / n)
        out[s] = np.tile(w, n // (2 * half))
    return out


@dataclass
class OraclePlan:
    """FftPlan(n, ModeSpec.mx(fmt, B)) restated: fftcore.py:93-117."""

    n: int
    fmt: Fmt
    block_size: int
    wcr: np.ndarray
    wci: np.ndarray
    ws: np.ndarray

    @property
    def stages(self):
        return self.n.bit_length() - 1

    @property
    def cpb(self):
        return min(self.block_size // 2, self.n // 2)


def make_plan(n: int, fmt, block_size: int = 32) -> OraclePlan:
    fmt = as_fmt(fmt)
    if n < 2 or n & (n - 1):
        raise ValueError(f"transform length must be a power of two >= 2, got {n}")
    tw = np.ascontiguousarray(ref_twiddles(n)).view(np.float64)
    cpb = min(block_size // 2, n // 2)
    st, m = n.bit_length() - 1, n // 2
    wcr = np.empty((st, m))
    wci = np.empty((st, m))
    ws = np.empty((st, m // cpb))
    lib().orc_encode_twiddles(_dp(tw), n, cpb, *fmt.args, _dp(wcr), _dp(wci), _dp(ws))
    return OraclePlan(n, fmt, block_size, wcr, wci, ws)


class _Dump(ctypes.Structure):
    _fields_ = [
        ("v_exp", ctypes.c_void_p),
        ("v_codes", ctypes.c_void_p),
        ("p_exp", ctypes.c_void_p),
        ("p_codes", ctypes.c_void_p),
        ("p_shift", ctypes.c_void_p),
        ("stage_out", ctypes.c_void_p),
    ]


def fft_batch(x, plan: OraclePlan, inverse: bool = False, dump: bool = False):
    """_fft_batch_mx, fftcore.py:259-282 on a (batch, n) array -> complex64.
    With dump=True also returns the per-stage capture dict (arrays [stage][batch]...)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if x.ndim == 1:
        x = x[None]
    b, n = x.shape
    assert n == plan.n
    y = np.empty((b, n), dtype=np.complex64)
    d = None
    cap = None
    if dump:
        st, m = plan.stages, n // 2
        nb = m // plan.cpb
        cap = dict(
            v_exp=np.zeros((st, b, nb), np.int32),
            v_codes=np.zeros((st, b, m, 2)),
            p_exp=np.zeros((st, b, nb), np.int32),
            p_codes=np.zeros((st, b, m, 2)),
            p_shift=np.zeros((st, b, nb), np.int32),
            stage_out=np.zeros((st, b, n), np.complex64),
        )
        d = _Dump(*(cap[k].ctypes.data for k in ("v_exp", "v_codes", "p_exp", "p_codes",
                                                  "p_shift", "stage_out")))
    xv = x.view(np.float64)
    rc = lib().orc_fft_batch_mx(
        _dp(xv), b, n, plan.block_size, *plan.fmt.args, _dp(plan.wcr), _dp(plan.wci),
        _dp(plan.ws), int(inverse), _fp(y.view(np.float32)),
        ctypes.cast(ctypes.pointer(d), ctypes.c_void_p) if d is not None else None,
    )
    if rc:
        raise MemoryError("oracle allocation failed")
    return (y, cap) if dump else y


def fft2(x, plan: OraclePlan, inverse: bool = False) -> np.ndarray:
    """fft_2d, fftcore.py:344-353 -> complex64 (n, n)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    n = plan.n
    assert x.shape == (n, n)
    y = np.empty((n, n), dtype=np.complex64)
    rc = lib().orc_fft2_mx(_dp(x.view(np.float64)), n, plan.block_size, *plan.fmt.args,
                           _dp(plan.wcr), _dp(plan.wci), _dp(plan.ws), int(inverse),
                           _fp(y.view(np.float32)))
    if rc:
        raise MemoryError("oracle allocation failed")
    return y


@dataclass(frozen=True)
class PrescaleOut:
    k: int
    a_max: float
    p_tau: float
    k1: int
    k2: int


def compute_prescale(x, target=1.0, tau=1.0, tau_min=2.0**-20, k_min=-40, k_max=40):
    """compute_prescale, prescale.py:61-73."""
    x = np.asarray(x)
    is_c = np.iscomplexobj(x)
    a = np.ascontiguousarray(x, dtype=np.complex128 if is_c else np.float64)
    flat = a.reshape(-1)
    am, pt = ctypes.c_double(), ctypes.c_double()
    k1, k2, k = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    rc = lib().orc_compute_prescale(
        _dp(flat.view(np.float64)), flat.size, int(is_c), target, tau, tau_min, k_min, k_max,
        ctypes.byref(am), ctypes.byref(pt), ctypes.byref(k1), ctypes.byref(k2), ctypes.byref(k))
    if rc:
        raise ValueError("non-finite input to prescale")
    return PrescaleOut(k.value, am.value, pt.value, k1.value, k2.value)


def pipeline(x, plan: OraclePlan, roundtrip: bool, target=1.0, tau=1.0, tau_min=2.0**-20,
             k_min=-40, k_max=40):
    """forward_pipeline / roundtrip_pipeline, mri.py:84-107, for one (C, n, n) stack.
    Returns (complex128 per-coil output after undo, RSS FP64 (n, n), k)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    if x.ndim == 2:
        x = x[None]
    c, n, _ = x.shape
    out = np.empty_like(x)
    rss = np.empty((n, n))
    k = ctypes.c_int()
    rc = lib().orc_pipeline(_dp(x.view(np.float64)), c, n, plan.block_size, *plan.fmt.args,
                            _dp(plan.wcr), _dp(plan.wci), _dp(plan.ws), target, tau, tau_min,
                            k_min, k_max, int(roundtrip), _dp(out.view(np.float64)), _dp(rss),
                            ctypes.byref(k))
    if rc:
        raise ValueError("oracle pipeline failed (non-finite input or allocation)")
    return out, rss, k.value


def cabs(x) -> np.ndarray:
    """np.abs(complex128) as restated in C (numpy 2.3.5 SIMD formula)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.complex128))
    out = np.empty(x.shape)
    lib().orc_cabs(_dp(x.view(np.float64)), x.size, _dp(out))
    return out


def psnr(ref, test) -> float:
    """metrics.py:38-47 (host scoring helper)."""
    r = np.asarray(ref, dtype=np.float64)
    t = np.asarray(test, dtype=np.float64)
    mse = float(np.mean((r - t) ** 2))
    if mse == 0.0:
        return math.inf
    return 20.0 * math.log10(float(r.max()) / math.sqrt(mse))


def nmse(ref, test) -> float:
    """metrics.py:50-56 (host scoring helper)."""
    r = np.asarray(ref, dtype=np.float64)
    t = np.asarray(test, dtype=np.float64)
    return float(np.sum((r - t) ** 2)) / float(np.sum(r**2))


def reference_fft2_f64(x, inverse: bool = False) -> np.ndarray:
    """FP64 reference-mode 2-D transform (fftcore.py:243-256 composed as fft_2d):
    the accuracy yardstick for PSNR scoring, via the same radix-2 DIT in FP64."""
    x = np.asarray(x, dtype=np.complex128)
    n = x.shape[-1]
    tw = ref_twiddles(n)
    bits = n.bit_length() - 1
    perm = np.array([int(format(i, f"0{bits}b")[::-1], 2) if bits else 0 for i in range(n)])

    def batch(a):
        y = a[:, perm].astype(np.complex128)
        b = y.shape[0]
        for s in range(bits):
            half = 1 << s
            w = tw[s]
            if inverse:
                w = np.conj(w)
            view = y.reshape(b, -1, 2 * half)
            u = view[..., :half]
            v = view[..., half:]
            t = v * w.reshape(-1, half)
            y = np.concatenate((u + t, u - t), axis=-1).reshape(b, n)
        return y

    rows = batch(x)
    cols = batch(np.ascontiguousarray(rows.T))
    return np.asarray(cols.T, dtype=np.complex128)
