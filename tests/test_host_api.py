"""Host-side parts of the API that need no GPU: coil maps, MXCG grid files
(byte-identical to the reference's writer, tests/golden/phantoms.npz), the
reference's error behaviour, and the full export list."""

import os
import re

import numpy as np
import pytest

import paper_2512_04317_b200 as mx
from conftest import golden


def test_exports_cover_reference_api():
    ref = os.path.join(os.path.dirname(__file__), "golden", "reference_exports.txt")
    names = open(ref).read().split()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(mx, n)]
    assert not missing, missing


def test_coil_sensitivities_match_reference():
    g = golden("phantoms")
    assert np.array_equal(mx.coil_sensitivities(16, 4, 3), g["sens"])


def test_mxcg_write_read_roundtrip_and_bytes(tmp_path):
    g = golden("phantoms")
    for ci, case in enumerate(g["cases"]):
        ksp = mx.ComplexGrid(g[f"c{ci}_ksp"], "kspace")
        p = tmp_path / f"g{ci}.mxcg"
        mx.write_grid(ksp, p)
        assert p.read_bytes() == g[f"c{ci}_mxcg"].tobytes(), case
        back = mx.read_grid(p)
        assert back.domain == "kspace" and np.array_equal(back.data, ksp.data)
    img = mx.ComplexGrid(g["c0_img"], "image")
    mx.write_grid(img, tmp_path / "i.mxcg")
    assert mx.read_grid(tmp_path / "i.mxcg").domain == "image"


def test_mxcg_errors(tmp_path):
    g = golden("phantoms")
    good = g["c2_mxcg"].tobytes()
    cases = [(b"XX", mx.BadMagic), (b"MXCG", mx.TruncatedFile), (b"NOPE" + good[4:], mx.BadMagic),
             (good[:4] + (2).to_bytes(4, "little") + good[8:], mx.BadVersion),
             (good[:8] + bytes([7]) + good[9:], mx.FileFormatError), (good[:-8], mx.TruncatedFile),
             (good + b"\0", mx.FileFormatError)]
    nan = bytearray(good)
    nan[17:25] = np.array([np.nan]).tobytes()
    cases.append((bytes(nan), mx.NonFinitePayload))
    for i, (blob, exc) in enumerate(cases):
        p = tmp_path / f"bad{i}.mxcg"
        p.write_bytes(blob)
        with pytest.raises(exc):
            mx.read_grid(p)


def test_phantom_config_errors():
    with pytest.raises(mx.ConfigError):
        mx.gen_phantom(12, 1, 0)
    with pytest.raises(mx.ConfigError):
        mx.gen_phantom(16, 0, 0)
