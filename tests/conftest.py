"""Shared fixtures.  The CPU oracle (oracle/) is the checker; tests marked
``gpu`` exercise the CUDA product through its C-ABI on a B200."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def rng():
    # same seed as the reference suite's session rng (reference tests/conftest.py:60-62)
    return np.random.default_rng(20240817)


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def digest(a) -> str:
    """SHA-256 of an array's values, -0.0 folded into +0.0 (the same helper as
    tests/golden/make_golden.py; the bigshapes fixture pins large reference
    outputs by digest)."""
    import hashlib

    a = np.ascontiguousarray(np.asarray(a) + 0.0)
    return hashlib.sha256(a.tobytes()).hexdigest()


def bigshape_cases():
    """(key, tag, fmt, block, image index) of the pipeline cases in bigshapes.npz."""
    g = golden("bigshapes")
    out = []
    for key in g["cases"]:
        key = str(key)
        if key.startswith("c5_"):
            continue
        tag, fmt, b, i = key.split("_")
        out.append((key, tag, fmt, int(b[1:]), int(i[1:])))
    return out


def bigshape_image(tag, i):
    from paper_2512_04317_b200.workloads import ellipse_kspace

    if tag == "c3":
        return ellipse_kspace(512, seed=501, noise=0.01)
    return ellipse_kspace(128, seed=601 + i, noise=0.05)
