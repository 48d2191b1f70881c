"""MXCG grid files (the reference's interchange format, mri.py:196-239):
a 17-byte little-endian header -- magic b"MXCG", uint32 version 1, uint8
domain (0 k-space, 1 image), uint32 coils, uint32 n -- followed by
coils * n * n complex128 values.  Host-side I/O, same errors as the reference."""

from __future__ import annotations

import struct

import numpy as np

from .errors import BadMagic, BadVersion, FileFormatError, NonFinitePayload, TruncatedFile

MAGIC = b"MXCG"
VERSION = 1
_HDR = struct.Struct("<4sIBII")


def write_grid(grid, path) -> None:
    from .mri import KSPACE

    head = _HDR.pack(MAGIC, VERSION, 0 if grid.domain == KSPACE else 1, grid.coils, grid.n)
    body = np.ascontiguousarray(grid.data, dtype="<c16").tobytes()
    with open(path, "wb") as f:
        f.write(head + body)


def read_grid(path):
    from .mri import IMAGE, KSPACE, ComplexGrid

    with open(path, "rb") as f:
        blob = f.read()
    if len(blob) < _HDR.size:
        if blob[:4] != MAGIC:
            raise BadMagic("not an MXCG file")
        raise TruncatedFile("incomplete MXCG header")
    magic, version, domain, coils, n = _HDR.unpack_from(blob)
    if magic != MAGIC:
        raise BadMagic(f"bad magic {magic!r}")
    if version != VERSION:
        raise BadVersion(f"unsupported MXCG version {version}")
    if domain not in (0, 1):
        raise FileFormatError(f"unknown domain code {domain}")
    need = coils * n * n * 16
    body = blob[_HDR.size:]
    if len(body) < need:
        raise TruncatedFile(f"expected {need} payload bytes, got {len(body)}")
    if len(body) > need:
        raise FileFormatError(f"{len(body) - need} trailing bytes")
    data = np.frombuffer(body, dtype="<c16").reshape(coils, n, n)
    if not np.isfinite(data).all():
        raise NonFinitePayload("non-finite values in MXCG payload")
    return ComplexGrid(data.astype(np.complex128), KSPACE if domain == 0 else IMAGE)
