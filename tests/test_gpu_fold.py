"""The prescale statistics folded into the first transform pass
(mxfft_pipeline_folded: compute_prescale, prescale.py:61-73, riding on the
first row pass of fft_2d, fftcore.py:344-353) against the standard path
(statistics kernels + mxfft_fft2) and the oracle.  Settled stacks must be
bit-identical; stacks the in-kernel proofs cannot settle must be flagged and
come out identical after pipeline_resolve."""
import math

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


def _rows(mx, res):
    from paper_2512_04317_b200.prescale import decode_results

    return decode_results(res)


def _same(torch, a, b):
    return torch.equal(torch.view_as_real(a), torch.view_as_real(b))


@pytest.mark.parametrize("n,batch,noise", [(128, 41, 0.05), (256, 7, 0.01), (512, 3, 0.01)])
@pytest.mark.parametrize("fmt,bsz", [("e4m3", 32), ("e5m2", 32), ("e3m2", 16), ("e2m3", 64), ("e2m1", 32)])
@pytest.mark.parametrize("roundtrip", [False, True])
def test_fold_equals_standard(mx, torch, n, batch, noise, fmt, bsz, roundtrip):
    """BASELINE-style k-space (phantom + noise): every stack is settled in the
    first pass (flags == 8), k and every output bit equal the standard path."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=4000 + n + bsz, noise=noise)).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    cfg = mx.PrescaleConfig()
    assert mx.mri.folded_pipeline_supported(p)
    y0, k0, r0 = mx.pipeline_device(x, p, cfg, roundtrip, fold=False, fused=False)
    y1, k1, r1 = mx.pipeline_device(x, p, cfg, roundtrip, fold=True, fused=False)
    rows = _rows(mx, r1)
    assert (rows["flags"] == 8).all(), rows["flags"]
    assert torch.equal(k0, k1)
    assert _same(torch, y0, y1)
    full = _rows(mx, r0)
    assert (rows["k1"] == full["k1"]).all()
    assert np.allclose(rows["a_max"], full["a_max"], rtol=1e-6, atol=0)
    assert mx.pipeline_resolve(x, y1, k1, r1, p, cfg, roundtrip) == 0


def test_fold_vs_oracle_and_repeatable(mx, torch):
    """folded C4-shaped batch against the oracle, and identical on a second call
    into the same buffers (accumulators re-zeroed)"""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    n, batch = 128, 6
    xh = ellipse_kspace_batch(batch, n, seed=77, noise=0.05)
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    op = O.make_plan(n, O.E4M3, 32)
    cfg = mx.PrescaleConfig()
    y = torch.empty_like(x)
    k = torch.empty(batch, dtype=torch.int32, device="cuda")
    for _ in range(2):
        y.zero_()
        _, _, res = mx.pipeline_device(x, p, cfg, True, out=y, k=k, fold=True, fused=False)
        assert (_rows(mx, res)["flags"] == 8).all()
        for i in range(batch):
            want, _, kw = O.pipeline(xh[i], op, True)
            assert int(k[i]) == kw
            assert np.array_equal(y[i].cpu().numpy().astype(np.complex128), want[0])


def test_fold_multicoil_shares_one_k(mx, torch):
    """stacks of 4 coils share one prescale: folded == standard"""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    n, coils, stacks = 128, 4, 5
    xh = ellipse_kspace_batch(coils * stacks, n, seed=91, noise=0.02)
    xh *= np.linspace(0.3, 7.0, coils * stacks, dtype=np.float32)[:, None, None]  # coils of unequal gain
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    y0, k0, _ = mx.pipeline_device(x, p, cfg, True, coils=coils, fold=False, fused=False)
    y1, k1, r1 = mx.pipeline_device(x, p, cfg, True, coils=coils, fold=True, fused=False)
    assert k1.numel() == stacks and torch.equal(k0, k1)
    assert (_rows(mx, r1)["flags"] == 8).all()
    assert _same(torch, y0, y1)


def test_fold_unsettled_stacks_are_flagged_and_resolved(mx, torch):
    """Inputs on which a proof fails: many tiny nonzero magnitudes (k2 exceeds
    k1), a peak on a log2 rounding boundary, magnitudes near the ends of FP32's
    range (block exponents near their clamps), an all-zero image (settled by
    the reference's own formula).  Flagged stacks equal the standard path after
    pipeline_resolve; settled neighbours are untouched."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    n = 256
    xh = ellipse_kspace_batch(8, n, seed=5, noise=0.01)
    xh[1, :64, :] = 1e-9 * (1 + 1j)          # a quarter of the points tiny: k2 > k1, the counting proof fails
    xh[7, 17, 33] = 1e-9 * (1 + 1j)          # ONE tiny value does not move the 1st percentile: still settled
    peak = np.abs(xh[2]).max()
    xh[2] *= np.float32(np.sqrt(2.0) / peak)  # a_max ~ sqrt(2): log2(1 / a_max) ~ -0.5
    xh[3] *= np.float32(1e-30)               # tiny magnitudes
    xh[4] *= np.float32(1e+25)               # huge magnitudes (keys overflow FP32)
    xh[5] = 0                                # all zeros
    xh[6, :, :] = 0
    xh[6, 3, 4] = 2.5 - 1j                   # a single nonzero point
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    for roundtrip in (False, True):
        y0, k0, r0 = mx.pipeline_device(x, p, cfg, roundtrip, fold=False, fused=False)
        assert mx.pipeline_resolve(x, y0, k0, r0, p, cfg, roundtrip) == 0
        y1, k1, r1 = mx.pipeline_device(x, p, cfg, roundtrip, fold=True, fused=False)
        flags = _rows(mx, r1)["flags"].copy()
        assert flags[0] == 8 and flags[7] == 8
        assert flags[1] == 4 and flags[3] == 4 and flags[4] == 4, flags
        assert flags[5] in (0, 2)  # all zeros: the formula itself
        settled = [i for i in range(8) if not flags[i] & 4]
        for i in settled:
            assert int(k1[i]) == int(k0[i]) and _same(torch, y0[i], y1[i]), i
        nredo = mx.pipeline_resolve(x, y1, k1, r1, p, cfg, roundtrip)
        assert nredo == int((flags & 4 != 0).sum())
        assert torch.equal(k0, k1)
        assert _same(torch, y0, y1)
        assert not (_rows(mx, r1)["flags"] & 4).any()


def test_fold_nonfinite_raises_in_resolve(mx, torch):
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    n = 128
    xh = ellipse_kspace_batch(3, n, seed=9, noise=0.05)
    xh[1, 5, 5] = np.nan
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    y, k, res = mx.pipeline_device(x, p, cfg, True, fold=True, fused=False)
    assert _rows(mx, res)["flags"][1] == 4
    with pytest.raises(mx.InvalidValue):
        mx.pipeline_resolve(x, y, k, res, p, cfg, True)


def test_fold_custom_config_where_k2_wins(mx, torch):
    """a tau_min large enough that k2 > k1: the fold must flag, never settle wrongly"""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    n = 128
    xh = ellipse_kspace_batch(4, n, seed=11, noise=0.05)
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E5M2, 32))
    cfg = mx.PrescaleConfig(tau_min=0.5)
    y0, k0, r0 = mx.pipeline_device(x, p, cfg, True, fold=False, fused=False)
    full = _rows(mx, r0)
    assert (full["k2"] > full["k1"]).all()
    y1, k1, r1 = mx.pipeline_device(x, p, cfg, True, fold=True, fused=False)
    assert (_rows(mx, r1)["flags"] == 4).all()
    assert mx.pipeline_resolve(x, y1, k1, r1, p, cfg, True) == 4
    assert torch.equal(k0, k1) and _same(torch, y0, y1)
    # the resolve has noted that the fold does not pay for this plan and configuration: the next
    # default call goes straight to the statistics kernels (full rows, nothing to resolve)
    y2, k2, r2 = mx.pipeline_device(x, p, cfg, True, fused=False)
    assert not (_rows(mx, r2)["flags"] & (4 | 8)).any()
    assert torch.equal(k0, k2) and _same(torch, y0, y2)


@pytest.mark.parametrize("graph", [False, True])
def test_fold_pipeline_host_resolves_unsettled_stacks(mx, torch, graph):
    """pipeline_host (H2D / folded pipeline / D2H slices): a stack the fold
    flags is redone from the host copy; the result equals the statistics-kernel
    path on every stack; non-finite input still raises"""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    n = 128
    xh = ellipse_kspace_batch(20, n, seed=21, noise=0.05)
    xh[3, :40, :] = 1e-9 * (1 + 1j)   # k2 > k1: unsettled by the fold
    xh[11] *= np.float32(1e-30)       # exponents outside the proven range
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    want, kw, rw = mx.pipeline_device(torch.from_numpy(xh).cuda(), p, cfg, True, fold=False, fused=False)
    assert mx.pipeline_resolve(torch.from_numpy(xh).cuda(), want, kw, rw, p, cfg, True) == 0
    h = torch.from_numpy(xh).pin_memory()
    out = torch.empty(h.shape, dtype=h.dtype).pin_memory()
    for _ in range(2):  # (graph=True: capture, then replay)
        out.zero_()
        got = mx.pipeline_host(h, p, cfg, True, out_host=out, chunks=3, graph=graph)
        assert _same(torch, got, want.cpu())
    xh[5, 0, 0] = np.inf
    with pytest.raises(mx.InvalidValue):
        mx.pipeline_host(torch.from_numpy(xh).pin_memory(), p, cfg, True, chunks=3, graph=graph)


def test_fold_c5_full_size_equals_standard(mx, torch):
    """C5: one 16384^2 image.  The folded pipeline (evidence gathered by the
    8192-point half-row kernel of the first split pass, grid-wide resolve,
    x 2^k at the load of that pass's last-stage kernel) equals the statistics
    kernels + mxfft_fft2 bit for bit, forward and round trip, and equals the
    exact global prescale's k."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    n = 16384
    x = ellipse_kspace_device(n, 7, noise=0.01)[None]
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    assert mx.mri.folded_pipeline_supported(p)
    kg = mx.compute_prescale_global(x[0], cfg).k
    for roundtrip in (False, True):
        y1, k1, r1 = mx.pipeline_device(x, p, cfg, roundtrip, fold=True)
        row = _rows(mx, r1)[0]
        assert int(row["flags"]) == 8 and int(k1[0]) == kg and int(row["nnz"]) == n * n
        y0 = mx.fft2_device(x, p, "roundtrip" if roundtrip else "forward", k=k1)
        assert _same(torch, y0, y1)
        del y0, y1
        torch.cuda.empty_cache()
    # a quarter of the image tiny: k2 wins, the fold must decline
    x[0, :4096] *= 1e-12
    _, _, r2 = mx.pipeline_device(x, p, cfg, False, fold=True)
    assert int(_rows(mx, r2)[0]["flags"]) == 4


@pytest.mark.parametrize("G", [2, 4])
def test_fold_slab_pipeline_threads_c5(mx, torch, G):
    """pipeline_slab with the folded prescale (first row pass with evidence, two
    small all-reduces, one read-back), G ranks as threads on one GPU at the
    C5 size: every rank's slab equals the single-GPU pipeline, k included; a
    slab pipeline without the fold gives the same bits."""
    import threading

    from paper_2512_04317_b200 import distributed as D
    from paper_2512_04317_b200.workloads import ellipse_kspace_device
    from test_gpu_r2 import ThreadComm

    n = 16384
    x = ellipse_kspace_device(n, 7, noise=0.01)
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    want, kw, _ = mx.pipeline_device(x[None], p, cfg, False)
    torch.cuda.synchronize()
    shared = {"world": G, "bar": threading.Barrier(G), "box": [None] * G}
    out = [None] * G
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                r0, r1 = D.shard_range(n, r, G)
                y, res = D.pipeline_slab(x[r0:r1], p, cfg, False, comm=ThreadComm(shared, r), fold=True)
                assert math.isnan(res.p_tau)  # the folded path (k-only), not the statistics fallback
                torch.cuda.current_stream().synchronize()
                out[r] = (torch.equal(torch.view_as_real(y), torch.view_as_real(want[0, r0:r1])), res.k)
        except BaseException as e:  # surface any rank's failure
            errs.append(e)
            shared["bar"].abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs[0]
    assert all(k == int(kw[0]) for _, k in out)
    assert all(ok for ok, _ in out)


@pytest.mark.parametrize("fmt,bsz,n", [("e4m3", 32, 128), ("e5m2", 16, 128), ("e2m1", 64, 256), ("e3m2", 32, 512)])
def test_fold_randomized_against_standard(mx, torch, fmt, bsz, n):
    """Randomized stress of the fold's proofs: images with random power-of-two
    gains over 2^+-70, random fractions of exact zeros, sparse images, heavy
    tails, isolated and clustered tiny values, constant images.  Whatever the
    fold settles must equal the statistics path bit for bit (k and outputs);
    whatever it declines must do so after pipeline_resolve; nothing else may
    happen."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    import os

    soak = int(os.environ.get("MXFFT_FOLD_SOAK", "0"))  # other seeds for soak runs (tools/fold_soak.sh)
    rng = np.random.default_rng(1234 + n + bsz + 1000 * soak)
    batch = 96 if n == 128 else 24
    xh = ellipse_kspace_batch(batch, n, seed=600 + n + 7919 * soak, noise=0.02)
    for i in range(batch):
        kind = i % 8
        if kind == 1:
            xh[i] *= np.float32(2.0 ** rng.integers(-70, 70))
        elif kind == 2:
            xh[i][rng.random((n, n)) < rng.uniform(0.0, 0.99)] = 0
        elif kind == 3:
            xh[i] = 0
            idx = rng.integers(0, n, (rng.integers(1, 40), 2))
            xh[i][idx[:, 0], idx[:, 1]] = (rng.standard_normal(len(idx)) + 1j * rng.standard_normal(len(idx))).astype(np.complex64)
        elif kind == 4:
            xh[i] = ((rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
                     * 10.0 ** rng.uniform(-6, 6, (n, n))).astype(np.complex64)
        elif kind == 5:
            m = rng.random((n, n)) < rng.choice([1e-4, 1e-3, 0.02, 0.3])
            xh[i][m] *= np.float32(1e-12)
        elif kind == 6:
            xh[i] = np.complex64(complex(rng.uniform(-3, 3), rng.uniform(-3, 3))) * np.float32(2.0 ** rng.integers(-20, 20))
        elif kind == 7:
            xh[i, : n // 2] *= np.float32(2.0 ** -rng.integers(10, 40))
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    cfg = mx.PrescaleConfig()
    for roundtrip in (False, True):
        y0, k0, r0 = mx.pipeline_device(x, p, cfg, roundtrip, fold=False, fused=False)
        assert mx.pipeline_resolve(x, y0, k0, r0, p, cfg, roundtrip) == 0
        y1, k1, r1 = mx.pipeline_device(x, p, cfg, roundtrip, fold=True, fused=False)
        flags = _rows(mx, r1)["flags"].copy()
        assert set(np.unique(flags & ~2)) <= {0, 4, 8}, np.unique(flags)
        for i in np.nonzero((flags & 4) == 0)[0]:
            assert int(k1[i]) == int(k0[i]), (i, i % 8)
            a, b = y1[i].cpu().numpy(), y0[i].cpu().numpy()
            assert ((a == b) | (np.isnan(a) & np.isnan(b))).all(), (i, i % 8)
        assert (flags[::8] == 8).all()  # the untouched phantoms are always settled
        mx.pipeline_resolve(x, y1, k1, r1, p, cfg, roundtrip)
        assert torch.equal(k0, k1)
        a, b = y1.cpu().numpy(), y0.cpu().numpy()
        assert ((a == b) | (np.isnan(a) & np.isnan(b))).all()
