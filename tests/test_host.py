"""CPU-side tests: the C-ABI library loads and exports every symbol the header
declares; host-side API logic (formats, modes, config validation, errors) that
runs before any device work."""

import math
import os
import re

import numpy as np
import pytest

import paper_2512_04317_b200 as mx
from paper_2512_04317_b200 import _native
from conftest import ROOT


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mxfft_b200.h")).read()
    return sorted(set(re.findall(r"\b(mxfft_[a-z0-9_]+)\s*\(", txt)))


def test_library_loads_and_exports_header():
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES), "ctypes signatures out of sync with the header"
    assert lib.mxfft_version() == 1


def test_library_is_sm100a_only():
    so = _native.LIB_PATH
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_sass_uses_hardware_minifloat_packs():
    import subprocess

    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun",
                           "_ZN5mxfft10k_mx_linesILi0ELi16ELb0ELi3EEEvNS_11MxLinesArgsE", _native.LIB_PATH],
                          capture_output=True, text=True).stdout
    assert "F2FP.SATFINITE.E4M3.F32.PACK_AB" in sass
    assert "F2FP.F16.E4M3.UNPACK_B" in sass


def test_no_gpu_means_loud_failure(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.quantize_array([1.0], mx.E4M3)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mx.make_plan(8, mx.ModeSpec.mx(mx.E4M3, 32))


class TestFormats:
    # reference tests/test_minifloat.py:28-57
    def test_constants(self):
        assert (mx.E4M3.max_finite, mx.E4M3.min_subnormal, mx.E4M3.emax) == (448.0, 2.0**-9, 8)
        assert (mx.E5M2.max_finite, mx.E5M2.emax) == (57344.0, 15)
        assert mx.E2M3.max_finite == 7.5 and mx.E3M2.max_finite == 28.0
        assert mx.FP16.max_finite == 65504.0 and mx.FP16.min_subnormal == 2.0**-24
        assert (mx.E2M1.max_finite, mx.E2M1.emax, mx.E2M1.min_subnormal) == (6.0, 2, 0.5)

    def test_registry(self):
        assert set(mx.FORMATS) == {"e4m3", "e5m2", "e2m3", "e3m2", "fp16"}
        assert mx.get_format("e4m3") is mx.E4M3
        with pytest.raises(KeyError, match="e5m2"):
            mx.get_format("nope")
        assert mx.get_mx_format("e2m1") is mx.E2M1

    def test_invalid(self):
        with pytest.raises(ValueError):
            mx.MinifloatFormat("bad", 1, 3)
        with pytest.raises(ValueError):
            mx.MinifloatFormat("bad", 4, 0)

    @pytest.mark.parametrize("f", [mx.E4M3, mx.E5M2, mx.E2M3, mx.E3M2, mx.FP16, mx.E2M1],
                             ids=lambda f: f.name)
    def test_enumerate(self, f):
        v = mx.enumerate_values(f)
        assert np.all(np.diff(v) > 0) and np.array_equal(v, -v[::-1])
        assert v[-1] == f.max_finite and v[v > 0][0] == f.min_subnormal

    def test_e4m3_count(self):
        assert mx.enumerate_values(mx.E4M3).size == 253
        assert mx.enumerate_values(mx.E2M1).size == 15


class TestModes:
    def test_from_name(self):
        # reference tests/test_fftcore.py:254-260
        assert mx.ModeSpec.from_name("reference").kind == "reference"
        assert mx.ModeSpec.from_name("fp16").kind == "fp16"
        m = mx.ModeSpec.from_name("e4m3", 8)
        assert m.kind == "mx" and m.fmt is mx.E4M3 and m.block_size == 8
        with pytest.raises(KeyError):
            mx.ModeSpec.from_name("e9m9")

    def test_block_size_validation(self):
        for b in (0, 1, 3, 7):
            with pytest.raises(ValueError):
                mx.ModeSpec.mx(mx.E4M3, b)

    def test_bad_sizes_rejected_before_device(self):
        for n in (0, 1, 3, 12, 100):
            with pytest.raises(mx.UnsupportedSize):
                mx.make_plan(n, mx.ModeSpec.reference())

    def test_reference_plan_twiddles(self):
        # reference tests/test_fftcore.py:33-41 (plan metadata is host-side)
        p = mx.make_plan(2, mx.ModeSpec.reference())
        assert np.array_equal(p.ref_twiddles[0], [1.0 + 0.0j])
        p = mx.make_plan(8, mx.ModeSpec.reference())
        assert abs(p.ref_twiddles[2][1] - math.sqrt(2) / 2 * (1 - 1j)) < 1e-15
        assert list(p.bitrev) == [0, 4, 2, 6, 1, 5, 3, 7]


class TestPrescaleConfig:
    def test_defaults(self):
        c = mx.PrescaleConfig()
        assert (c.target, c.tau, c.tau_min, c.k_min, c.k_max) == (1.0, 1.0, 2.0**-20, -40, 40)

    @pytest.mark.parametrize("kw", [dict(target=0.0), dict(tau=0.0), dict(tau=100.0),
                                    dict(tau_min=-1.0), dict(k_min=5, k_max=-5)])
    def test_rejects(self, kw):
        with pytest.raises(mx.ConfigError):
            mx.PrescaleConfig(**kw)

    def test_host_k_rule(self):
        from paper_2512_04317_b200.prescale import k_from_stats

        c = mx.PrescaleConfig()
        assert k_from_stats(8.0, 8.0, c)[0] == -3
        assert k_from_stats(1.0, 2.0**-30, c) == (10, 0, 10)
        assert k_from_stats(2.0**-60, 2.0**-60, c)[0] == 40


def test_grid_validation():
    with pytest.raises(mx.ShapeError):
        mx.ComplexGrid(np.ones((4, 4)), "image")
    with pytest.raises(mx.InvalidValue):
        mx.ComplexGrid(np.ones((1, 4, 4)), "spectral")
    bad = np.ones((1, 4, 4), dtype=complex)
    bad[0, 0, 0] = np.nan
    with pytest.raises(mx.InvalidValue):
        mx.ComplexGrid(bad, "image")


def test_error_hierarchy():
    for e in (mx.InvalidValue, mx.ShapeError, mx.UnsupportedSize, mx.MantissaOverflow,
              mx.ConfigError, mx.FileFormatError):
        assert issubclass(e, mx.MxfftError)
    assert issubclass(mx.BadMagic, mx.FileFormatError)
    assert mx.ConfigError("tau", "x").field == "tau"
