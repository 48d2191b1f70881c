"""The TMA line kernel (k_mx_lines_tma: n = 128 / 256 / 512 row passes stored
transposed, tile in by TMA tensor load, group out by one TMA tensor store)
against the per-thread copy-out kernel and the oracle (fftcore.py:344-353)."""
import numpy as np
import pytest

import oracle as O  # the checker (tests/conftest.py puts oracle/ on the path)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    import paper_2512_04317_b200 as m

    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


def _knobs(L, tma=1, fused=-1, pdl=1):
    L.mxfft_tma_store(tma)
    L.mxfft_fused_image(fused)
    L.mxfft_pdl(pdl)


@pytest.mark.parametrize("n,batch", [(128, 37), (256, 9), (512, 3)])
@pytest.mark.parametrize("fmt,bsz", [("e4m3", 32), ("e5m2", 16), ("e3m2", 64), ("e2m3", 32), ("e2m1", 16)])
def test_tma_kernel_equals_copy_out(mx, torch, n, batch, fmt, bsz):
    """every mode, with per-image k, out of place: identical bits with the TMA
    kernel on and off (and with programmatic dependent launch off)"""
    from paper_2512_04317_b200 import _native
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    L = _native.lib()
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=11 + n, noise=0.03)).cuda()
    kk = torch.arange(batch, dtype=torch.int32, device="cuda") % 9 - 4
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    try:
        for mode in ("forward", "inverse", "roundtrip"):
            _knobs(L, tma=0, fused=0)
            want = mx.fft2_device(x, p, mode, k=kk)
            torch.cuda.synchronize()
            for pdl in (1, 0):
                _knobs(L, tma=1, fused=0, pdl=pdl)
                got = mx.fft2_device(x, p, mode, k=kk)
                assert torch.equal(torch.view_as_real(got), torch.view_as_real(want)), (mode, pdl)
    finally:
        _knobs(L)


@pytest.mark.parametrize("n", [128, 256, 512])
def test_tma_kernel_vs_oracle_with_replayed_groups(mx, torch, n):
    """fft_2d against the oracle on a batch whose images span ordinary and
    extreme magnitudes: groups with a block outside the fast exponent range are
    replayed exactly and leave through the kernel's plain store loop"""
    from paper_2512_04317_b200 import _native

    L = _native.lib()
    rng = np.random.default_rng(n)
    scales = [1.0, 1e-38, 3e-3, 1e30, 1e-30, 7.0]
    x = np.stack([((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) * s).astype(np.complex64)
                  for s in scales])
    x[2, ::5] = 0
    x[4, :, 3::7] = 0
    op = O.make_plan(n, O.E4M3, 32)
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    try:
        _knobs(L, tma=1, fused=0)
        got = mx.fft2_device(torch.from_numpy(x).cuda(), p, "forward").cpu().numpy()
    finally:
        _knobs(L)
    for i in range(len(scales)):
        want = O.fft2(x[i], op).astype(np.complex64)
        same = (got[i] == want) | (np.isnan(got[i]) & np.isnan(want))
        assert same.all(), (n, scales[i], int((~same).sum()))


def test_tma_kernel_in_place_and_many_groups(mx, torch):
    """in place (x is y: pass 1 reads x, pass 2 writes it) and a batch with more
    groups than resident CTAs, walked in both directions (fft2 reverses pass 2)"""
    from paper_2512_04317_b200 import _native
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    L = _native.lib()
    x = torch.from_numpy(ellipse_kspace_batch(64, 256, seed=5)).cuda()
    p = mx.make_plan(256, mx.ModeSpec.mx(mx.E4M3, 32))
    try:
        _knobs(L, tma=0)
        want = mx.fft2_device(x, p, "roundtrip")
        torch.cuda.synchronize()
        _knobs(L, tma=1)
        y = x.clone()
        mx.fft2_device(y, p, "roundtrip", out=y)
        assert torch.equal(torch.view_as_real(y), torch.view_as_real(want))
    finally:
        _knobs(L)


@pytest.mark.parametrize("n,batch", [(128, 300), (256, 80), (512, 20)])
def test_tma_kernel_repeatable_under_buffer_reuse(mx, torch, n, batch):
    """the same input 20 times, with one CTA per SM (every CTA walks several
    groups: the tile / work buffers, the mbarrier phases and the split named
    barriers are reused many times) and with the default occupancy: identical
    bits every time (a missing wait between the TMA proxies and the threads'
    shared-memory accesses would show up as run-to-run differences)"""
    from paper_2512_04317_b200 import _native
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    L = _native.lib()
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=n, noise=0.02)).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    try:
        _knobs(L, tma=0, fused=0)
        want = mx.fft2_device(x, p, "roundtrip")
        torch.cuda.synchronize()
        _knobs(L, tma=1, fused=0)
        for per_sm in (1, 0):
            L.mxfft_lines_ctas_per_sm(per_sm)
            for it in range(20):
                got = mx.fft2_device(x, p, "roundtrip")
                assert torch.equal(torch.view_as_real(got), torch.view_as_real(want)), (per_sm, it)
    finally:
        L.mxfft_lines_ctas_per_sm(0)
        _knobs(L)


def test_tma_kernel_fewer_groups_than_ctas(mx, torch):
    """one image: fewer groups than resident CTAs (idle CTAs leave at once)"""
    from paper_2512_04317_b200 import _native

    L = _native.lib()
    rng = np.random.default_rng(3)
    for n in (128, 256, 512):
        x = (rng.standard_normal((1, n, n)) + 1j * rng.standard_normal((1, n, n))).astype(np.complex64)
        op = O.make_plan(n, O.E2M1, 16)
        p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format("e2m1"), 16))
        try:
            _knobs(L, tma=1, fused=0)
            got = mx.fft2_device(torch.from_numpy(x).cuda(), p, "forward").cpu().numpy()
        finally:
            _knobs(L)
        assert np.array_equal(got[0], O.fft2(x[0], op).astype(np.complex64)), n
