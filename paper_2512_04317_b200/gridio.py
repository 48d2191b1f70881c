"""TRANSCRIPTION, labelled as such: read_grid / write_grid follow the
reference's MXCG reader and writer (pkg/src/mxfft/mri.py:202-239) statement
by statement, including the error strings, because the file bytes and the
exceptions are the interface.  Host-only file I/O,
kept only so that the reference's public names resolve (drop-in
completeness); not part of the B200 hot path and claims no credit."""

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
