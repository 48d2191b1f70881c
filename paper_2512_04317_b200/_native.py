"""ctypes binding of the C-ABI library (include/mxfft_b200.h).

The product has no CPU fallback: importing a compute entry point without the
built ``_lib/libmxfft_b200.so`` or without a CUDA device raises immediately.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# MXFFT_B200_LIB: an alternative build of the same library (A/B profiling)
LIB_PATH = os.environ.get("MXFFT_B200_LIB") or os.path.join(_HERE, "_lib", "libmxfft_b200.so")

_lib = None


class FormatC(ctypes.Structure):
    _fields_ = [("exponent_bits", ctypes.c_int32), ("mantissa_bits", ctypes.c_int32),
                ("policy", ctypes.c_int32), ("bias", ctypes.c_int32)]


class PrescaleCfgC(ctypes.Structure):
    _fields_ = [("target", ctypes.c_double), ("tau", ctypes.c_double),
                ("tau_min", ctypes.c_double), ("k_min", ctypes.c_int32),
                ("k_max", ctypes.c_int32)]


# mxfft_prescale_result, as a numpy structured dtype (40 bytes, C layout)
PRESCALE_RESULT_DTYPE = np.dtype([("a_max", "<f8"), ("p_tau", "<f8"), ("k1", "<i4"),
                                  ("k2", "<i4"), ("k", "<i4"), ("flags", "<i4"),
                                  ("nnz", "<i8")])

# exported symbols and their signatures (argtypes, restype)
_vp, _i32, _i64, _u = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
_fp = ctypes.POINTER(FormatC)
SIGNATURES = {
    "mxfft_version": ([], _i32),
    "mxfft_last_error": ([], ctypes.c_char_p),
    "mxfft_launch_count": ([], _i64),
    "mxfft_profile_stage_limit": ([_i32], None),
    "mxfft_profile_flags": ([_i32], None),
    "mxfft_lines_ctas_per_sm": ([_i32], None),
    "mxfft_quantize_f64": ([_vp, _vp, _i64, _fp, _vp, _u], _i32),
    "mxfft_mx_encode_f64": ([_vp, _i64, _i32, _fp, _vp, _vp, _vp, _u], _i32),
    "mxfft_mx_decode_f64": ([_vp, _vp, _i64, _i32, _vp, _u], _i32),
    "mxfft_plan_create": ([ctypes.POINTER(_vp), _i32, _fp, _i32, _vp, _u], _i32),
    "mxfft_plan_destroy": ([_vp], _i32),
    "mxfft_plan_twiddles": ([_vp, _vp, _vp, _vp], _i32),
    "mxfft_fft_rows": ([_vp, _vp, _vp, _i64, _i32, _u], _i32),
    "mxfft_fft_rows_seg": ([_vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _u], _i32),
    "mxfft_fft_cols": ([_vp, _vp, _vp, _i64, _i32, _u], _i32),
    "mxfft_fft_rows_scaled": ([_vp, _vp, _vp, _i64, _i32, _i32, _i32, _u], _i32),
    "mxfft_fft2": ([_vp, _vp, _vp, _i64, _i32, _vp, _i32, _vp, _i64, _u], _i32),
    "mxfft_fft2_workspace_bytes": ([_vp, _i64], _i64),
    "mxfft_transpose_c64": ([_vp, _vp, _i64, _i32, _u], _i32),
    "mxfft_transpose_c64_strided": ([_vp, _i64, _i64, _vp, _i64, _i32, _u], _i32),
    "mxfft_metrics": ([_vp, _vp, _i64, _i64, _i32, _vp, ctypes.c_double, ctypes.c_double, _vp, _u], _i32),
    "mxfft_fft_rows_fp16": ([_vp, _i32, _vp, _i64, _i32, _vp, _i32, _vp, _u], _i32),
    "mxfft_fft_rows_f64": ([_vp, _vp, _i64, _i32, _vp, _i32, _u], _i32),
    "mxfft_prescale_stats": ([_vp, _i32, _i64, _i64, ctypes.POINTER(PrescaleCfgC), _vp, _vp,
                              _vp, _i64, _u], _i32),
    "mxfft_prescale_workspace_bytes": ([_i64, _i64], _i64),
    "mxfft_rss": ([_vp, _i32, _i64, _i32, _i64, _vp, _u], _i32),
    "mxfft_pipeline_fused_supported": ([_vp], _i32),
    "mxfft_fused_image": ([_i32], None),
    "mxfft_tma_store": ([_i32], None),
    "mxfft_pdl": ([_i32], None),
    "mxfft_split_last_stage": ([_i32], None),
    "mxfft_pipeline_fused": ([_vp, _vp, _vp, _i64, _i32, ctypes.POINTER(PrescaleCfgC), _vp, _vp, _u], _i32),
    "mxfft_pipeline_folded_supported": ([_vp], _i32),
    "mxfft_pipeline_folded_workspace_bytes": ([_vp, _i64, _i32], _i64),
    "mxfft_pipeline_folded": ([_vp, _vp, _vp, _i64, _i32, _i32, ctypes.POINTER(PrescaleCfgC), _vp, _vp, _vp, _i64,
                               _u], _i32),
    "mxfft_fold_words_bytes": ([_i64], _i64),
    "mxfft_fft_rows_evidence": ([_vp, _vp, _vp, _i64, _i32, _vp, _i64, _u], _i32),
    "mxfft_fold_reduce": ([_vp, _i64, ctypes.POINTER(PrescaleCfgC), _i32, _vp, _u], _i32),
    "mxfft_fold_finish": ([_vp, _i64, ctypes.POINTER(PrescaleCfgC), _vp, _vp, _u], _i32),
    "mxfft_rss_scaled": ([_vp, _i32, _i64, _i32, _i64, _vp, _i32, _i32, _vp, _u], _i32),
    "mxfft_prescale_apply_c128": ([_vp, _vp, _i64, _i64, _vp, _u], _i32),
    "mxfft_mx_multiply_f64": ([_vp, _vp, _vp, _vp, _i64, _i32, _i32, _fp, _vp, _vp, _vp, _vp, _vp, _u], _i32),
    "mxfft_scale": ([_vp, _vp, _i64, _i32, ctypes.c_double, _u], _i32),
    "mxfft_cabs": ([_vp, _i32, _i64, _vp, _u], _i32),
    "mxfft_prescale_sample_keys": ([_vp, _i64, _i64, _vp, _u], _i32),
    "mxfft_prescale_count_range": ([_vp, _i64, ctypes.c_float, ctypes.c_float, ctypes.c_float, _vp, _vp,
                                    _i64, _vp, _i64, _u], _i32),
    "mxfft_selftest_hw_quantizer": ([_fp, _vp, _vp, _u], _i32),
    "mxfft_fft_rows_debug": ([_vp, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _u], _i32),
}


def load():
    """Load the shared library (no CUDA needed just to load)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"CUDA extension not built: {LIB_PATH} is missing "
                "(run __graft_entry__.build() or `make -C paper_2512_04317_b200/csrc`)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (argt, rest) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argt
            fn.restype = rest
        _lib = L
    return _lib


def lib():
    """The library, for compute calls: also requires a CUDA device."""
    L = load()
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2512_04317_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return L


_STATUS = {
    1: errors.InvalidValue,
    2: errors.ShapeError,
    3: errors.UnsupportedSize,
    4: ValueError,
    5: RuntimeError,
    6: errors.MantissaOverflow,
}


def check(rc: int) -> None:
    if rc != 0:
        msg = load().mxfft_last_error().decode(errors="replace")
        raise _STATUS.get(rc, RuntimeError)(msg)


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def launch_count() -> int:
    return int(load().mxfft_launch_count())
