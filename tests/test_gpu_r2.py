"""GPU parity at the BASELINE configurations' own shapes, and the round-2
additions: reference-digest fixtures (C3 512^2 x 9 format/block pairs, C4
128^2 with 5% noise, C5 16384-point rows), the full 16384^2 round trip
(mxfft_fft2's split-transpose path), the multi-rank slab path run with the
real CUDA primitives on one GPU (a thread-backed communicator, G = 2/4/8),
the FP64 epilogue of the ComplexGrid pipelines at the edges of FP32's range,
and the error paths of the device pipeline."""

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
from conftest import bigshape_cases, bigshape_image, digest, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mx():
    import paper_2512_04317_b200 as m

    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t

    return t


# ---------------------------------------------------------------------------
# reference digests at the BASELINE shapes
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("case", bigshape_cases(), ids=lambda c: c[0])
def test_baseline_shapes_match_reference_digests(mx, torch, case):
    """pipeline_device (the benchmark path) and the public ComplexGrid
    pipelines reproduce the reference's own outputs bit for bit: per-coil
    complex outputs of forward / round trip, RSS images, k, a_max, p_tau."""
    key, tag, fmt, bsz, i = case
    g = golden("bigshapes")
    x = bigshape_image(tag, i)
    assert digest(x) == str(g[key + "_x"]), "input generator differs from the fixture's"
    n = x.shape[0]
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    cfg = mx.PrescaleConfig()
    xd = torch.from_numpy(x[None].copy()).cuda()
    yf, kf, rf = mx.pipeline_device(xd, p, cfg, roundtrip=False)
    yr, kr, rr = mx.pipeline_device(xd, p, cfg, roundtrip=True)
    assert mx.pipeline_resolve(xd, yr, kr, rr, p, cfg, True) == 0
    k, k1, k2 = g[key + "_k"].tolist()
    assert int(kf[0]) == int(kr[0]) == k
    # the default path folds the statistics into the first pass (k-only rows: flags 8, k1 exact,
    # a_max to 2^-23); the statistics kernels (fold=False) give the full row
    fr = mx.prescale.decode_results(rr)[0]
    assert int(fr["flags"]) == 8 and int(fr["k1"]) == k1 and int(fr["k"]) == k
    assert abs(float(fr["a_max"]) / g[key + "_stats"].tolist()[0] - 1.0) < 1e-6
    ys, ks, rs = mx.pipeline_device(xd, p, cfg, roundtrip=True, fold=False)
    assert int(ks[0]) == k and torch.equal(torch.view_as_real(ys), torch.view_as_real(yr))
    st = mx.prescale.decode_results(rs)[0]
    assert (int(st["k1"]), int(st["k2"])) == (k1, k2)
    assert [float(st["a_max"]), float(st["p_tau"])] == g[key + "_stats"].tolist()
    assert digest(yf[0].cpu().numpy().astype(np.complex128)) == str(g[key + "_fwd"])
    assert digest(yr[0].cpu().numpy().astype(np.complex128)) == str(g[key + "_rt"])
    fwd = mx.forward_pipeline(mx.ComplexGrid(x[None].astype(np.complex128), "kspace"), p, cfg)
    rt = mx.roundtrip_pipeline(mx.ComplexGrid(x[None].astype(np.complex128), "image"), p, cfg)
    assert digest(fwd.pixels) == str(g[key + "_fwd_rss"])
    assert digest(rt.pixels) == str(g[key + "_rt_rss"])
    psnr, nmse = g[key + "_quality"].tolist()
    ref = np.abs(x.astype(np.complex128))
    assert abs(mx.psnr(ref, rt.pixels) - psnr) <= 0.01
    assert abs(np.sqrt(mx.nmse(ref, rt.pixels)) - np.sqrt(nmse)) <= 1e-4


def test_c5_rows_match_reference_digests(mx, torch):
    g = golden("bigshapes")
    rows = torch.from_numpy(g["c5_rows_x"]).cuda()
    for fmt, bsz in (("e4m3", 32), ("e2m1", 64)):
        p = mx.make_plan(16384, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
        for inv, d in ((False, "forward"), (True, "inverse")):
            y = mx.fft_rows_device(rows, p, inv)
            assert digest(y.cpu().numpy()) == str(g[f"c5_{fmt}_b{bsz}_{d}"]), (fmt, d)


# ---------------------------------------------------------------------------
# C5: the full 16384^2 image through mxfft_fft2 (row passes + tiled transposes)
# ---------------------------------------------------------------------------
def _oracle_rows_sampled(y_in, y_out, rows, plan, inverse, exp_out=0):
    """Check rows `rows` of a GPU row pass (input y_in, output y_out, both
    CUDA) against the oracle, in threads (the C oracle releases the GIL)."""
    def one(r):
        a = y_in[r].cpu().numpy()[None]
        want = O.fft_batch(a, plan, inverse)[0]
        if exp_out:
            want = (want.astype(np.complex128) * 2.0**exp_out).astype(np.complex64)
        got = y_out[r].cpu().numpy()
        return r, bool(np.array_equal(got, want))

    with ThreadPoolExecutor(os.cpu_count() or 4) as ex:
        bad = [r for r, ok in ex.map(one, rows) if not ok]
    assert not bad, f"rows {bad[:8]} differ from the oracle"


def test_c5_full_size_roundtrip_vs_oracle(mx, torch):
    """The 16384^2 pipeline exactly as bench.py runs it (global prescale, then
    mxfft_fft2 forward / round trip with x 2^k and 2^-(k + 28) fused), against
    a pass-by-pass chain of row transforms and transposes that is itself
    checked row by row against the threaded C oracle (64 random rows per pass,
    every pass).  Equal k; the chain and mxfft_fft2 agree on every point."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    n = 16384
    x = ellipse_kspace_device(n, 7, noise=0.01)
    cfg = mx.PrescaleConfig()
    res = mx.compute_prescale_global(x, cfg)
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    op = O.make_plan(n, O.E4M3, 32)
    kt = torch.tensor([res.k], dtype=torch.int32, device="cuda")
    rng = np.random.default_rng(16384)
    for mode in ("forward", "roundtrip"):
        y = mx.fft2_device(x[None], p, mode, k=kt)[0]
        # the chain: rows(2^k x) -> T -> rows -> T [-> rows_inv -> T -> rows_inv x 2^-(k+28) -> T]
        dirs = [False, False] + ([True, True] if mode == "roundtrip" else [])
        cur = (x * (2.0 ** res.k)).contiguous()  # exact (normal range)
        for i, inv in enumerate(dirs):
            last = i == len(dirs) - 1
            e_out = (-res.k - (28 if mode == "roundtrip" else 0)) if last else 0
            nxt = mx.fft_rows_device(cur, p, inv)
            if e_out:
                nxt = nxt * (2.0 ** e_out)  # exact power-of-two scaling in FP32 (normal range)
            _oracle_rows_sampled(cur, nxt, sorted(rng.choice(n, 64, replace=False).tolist()), op, inv, e_out)
            cur = nxt.t().contiguous()
            del nxt
        assert torch.equal(cur, y), f"{mode}: mxfft_fft2 differs from the verified pass chain"
        del cur, y
        torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# multi-rank slab path with the real CUDA kernels: G ranks as threads on one GPU
# ---------------------------------------------------------------------------
class ThreadComm:
    """The distributed.Comm interface for G ranks that are threads of one
    process, each on its own CUDA stream: a collective is a barrier, a
    synchronize, device copies between the ranks' tensors, and a barrier.
    Test infrastructure only -- the product path uses torch.distributed."""

    def __init__(self, shared, rank):
        self.s = shared
        self.rank = rank
        self.world = shared["world"]

    def _exchange(self, t):
        import torch

        torch.cuda.current_stream().synchronize()
        self.s["box"][self.rank] = t
        self.s["bar"].wait()
        got = [self.s["box"][r].clone() for r in range(self.world)]
        torch.cuda.current_stream().synchronize()
        self.s["bar"].wait()
        return got

    def sum_(self, t):
        parts = self._exchange(t)
        t.copy_(sum(parts[1:], parts[0]))
        return t

    def max_(self, t):
        import torch

        parts = self._exchange(t)
        t.copy_(torch.stack(parts).max(0).values)
        return t

    def all_gather_cat(self, t):
        import torch

        return torch.cat(self._exchange(t))

    def all_to_all(self, out, inp):
        parts = self._exchange(inp)
        G = self.world
        for r in range(G):
            out[r].copy_(parts[r].reshape((G,) + tuple(inp.shape[1:]))[self.rank])
        return out


@pytest.mark.parametrize("n,G", [(1024, 2), (1024, 4), (1024, 8), (512, 8)])
def test_slab_pipeline_threads_real_kernels(mx, torch, n, G):
    """pipeline_slab (global prescale + row passes + all-to-all transposes) with
    CudaOps, G ranks as threads on one GPU: every rank's slab of the round
    trip equals the single-image oracle pipeline, bit for bit, with equal k."""
    from paper_2512_04317_b200 import distributed as D
    from paper_2512_04317_b200.workloads import ellipse_kspace

    x = ellipse_kspace(n, 11 + G, noise=0.01)
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    shared = {"world": G, "bar": threading.Barrier(G), "box": [None] * G}
    out = [None] * G
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                r0, r1 = D.shard_range(n, r, G)
                xs = torch.from_numpy(x[r0:r1].copy()).cuda()
                y, res = D.pipeline_slab(xs, p, cfg, True, comm=ThreadComm(shared, r))
                torch.cuda.current_stream().synchronize()
                out[r] = (y.cpu().numpy(), res.k)
        except BaseException as e:  # surface any rank's failure
            errs.append(e)
            shared["bar"].abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs[0]
    want, _, k_o = O.pipeline(x, O.make_plan(n, O.E4M3, 32), True)
    assert all(k == k_o for _, k in out)
    got = np.concatenate([o[0] for o in out]).astype(np.complex128)
    assert np.array_equal(got, want[0])


# ---------------------------------------------------------------------------
# ComplexGrid pipelines at the edges of FP32's range: the reference scales in
# FP64 before the complex64 cast and undoes in FP64 (prescale.py:76-91)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("scale,roundtrip", [(5e34, False), (1e-50, False), (1e-50, True), (3e31, True)])
def test_grid_pipelines_fp64_edges_match_oracle(mx, scale, roundtrip):
    from paper_2512_04317_b200.workloads import ellipse_kspace

    x = ellipse_kspace(64, 21, noise=0.02).astype(np.complex128) * scale
    p = mx.make_plan(64, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    out_o, rss_o, k_o = O.pipeline(x, O.make_plan(64, O.E4M3, 32), roundtrip)
    grid = mx.ComplexGrid(x[None], "image" if roundtrip else "kspace")
    got = (mx.roundtrip_pipeline if roundtrip else mx.forward_pipeline)(grid, p, cfg).pixels
    assert np.isfinite(got).all()
    assert np.array_equal(got, rss_o)


def test_apply_prescale_dtypes_match_numpy(mx):
    import math

    rng = np.random.default_rng(3)
    arrays = [rng.standard_normal(37).astype(np.float32), rng.standard_normal(37),
              (rng.standard_normal(19) + 1j * rng.standard_normal(19)).astype(np.complex64),
              rng.standard_normal(19) + 1j * rng.standard_normal(19), np.arange(9, dtype=np.int32),
              rng.standard_normal(8).astype(np.float16)]
    with np.errstate(over="ignore"):
        for a in arrays:
            for k in (-140, -30, 0, 7, 130, 300):
                want = a * math.ldexp(1.0, k)
                got = mx.apply_prescale(a, k)
                assert got.dtype == want.dtype, (a.dtype, k)
                assert np.array_equal(got, want, equal_nan=True), (a.dtype, k)
                assert np.array_equal(mx.undo_prescale(got, k), want * math.ldexp(1.0, -k), equal_nan=True)


def test_rss_scaled_and_prescale_apply_kernels(mx, torch):
    from paper_2512_04317_b200 import _native

    L = _native.lib()
    rng = np.random.default_rng(4)
    x = (rng.standard_normal((2, 3, 50)) + 1j * rng.standard_normal((2, 3, 50))).astype(np.complex64)
    k = torch.tensor([5, -70], dtype=torch.int32, device="cuda")
    xd = torch.from_numpy(x).cuda()
    out = torch.empty((2, 50), dtype=torch.float64, device="cuda")
    _native.check(L.mxfft_rss_scaled(xd.data_ptr(), 0, 2, 3, 50, k.data_ptr(), -1, -8, out.data_ptr(),
                                     _native.stream_handle()))
    want = np.sqrt((np.abs(x.astype(np.complex128) * 2.0 ** np.array([-13, 62])[:, None, None]) ** 2).sum(1))
    assert np.array_equal(out.cpu().numpy(), want)
    x128 = rng.standard_normal((2, 64)) * 1e-40 + 1j * rng.standard_normal((2, 64)) * 1e30
    kk = torch.tensor([40, -20], dtype=torch.int32, device="cuda")
    y = torch.empty((2, 64), dtype=torch.complex64, device="cuda")
    xd = torch.from_numpy(x128).cuda()
    _native.check(L.mxfft_prescale_apply_c128(xd.data_ptr(), y.data_ptr(), 2, 64, kk.data_ptr(),
                                              _native.stream_handle()))
    with np.errstate(over="ignore"):
        want = (x128 * 2.0 ** np.array([40, -20])[:, None]).astype(np.complex64)
    assert np.array_equal(y.cpu().numpy(), want)


# ---------------------------------------------------------------------------
# device pipeline error paths (flags instead of host syncs)
# ---------------------------------------------------------------------------
def test_pipeline_device_shape_checks_and_nonfinite(mx, torch):
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    p = mx.make_plan(64, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    x = torch.from_numpy(ellipse_kspace_batch(3, 64, seed=5)).cuda()
    with pytest.raises(mx.ShapeError):
        mx.pipeline_device(x, p, cfg, True, coils=2)
    with pytest.raises(mx.ShapeError):
        mx.fft2_device(x, p, "forward", k=torch.zeros(2, dtype=torch.int32, device="cuda"))
    x[1, 3, 5] = float("nan")
    y, k, res = mx.pipeline_device(x, p, cfg, True)
    with pytest.raises(mx.InvalidValue):
        mx.pipeline_resolve(x, y, k, res, p, cfg, True)
    h = x.cpu().pin_memory()
    with pytest.raises(mx.InvalidValue):
        mx.pipeline_host(h, p, cfg, True, graph=False)


# ---------------------------------------------------------------------------
# the fused small-image kernel (mxfft_pipeline_fused, one 128^2 image per CTA)
# ---------------------------------------------------------------------------
def _fused_vs_unfused(mx, torch, x, fmt, bsz, roundtrip):
    p = mx.make_plan(128, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    assert mx.fused_pipeline_supported(p)
    cfg = mx.PrescaleConfig()
    xd = torch.from_numpy(x).cuda()
    from paper_2512_04317_b200 import _native

    y1, k1, r1 = mx.pipeline_device(xd, p, cfg, roundtrip, fused=True)
    _native.lib().mxfft_fused_image(0)  # the reference path: statistics kernel + four line passes
    try:
        y0, k0, r0 = mx.pipeline_device(xd, p, cfg, roundtrip, fused=False, fold=False)
        torch.cuda.synchronize()
        _native.lib().mxfft_fused_image(1)
        y2, k2, r2 = mx.pipeline_device(xd, p, cfg, roundtrip, fused=False, fold=False)  # statistics + fused fft2
        torch.cuda.synchronize()
    finally:
        _native.lib().mxfft_fused_image(-1)  # back to the automatic choice
    assert torch.equal(k2, k0) and torch.equal(r2, r0)
    a2, b2 = y2.cpu().numpy(), y0.cpu().numpy()
    assert ((a2 == b2) | (np.isnan(a2) & np.isnan(b2))).all()
    assert torch.equal(k1, k0)
    d1, d0 = mx.prescale.decode_results(r1), mx.prescale.decode_results(r0)
    ok = (d0["flags"] & 1) == 0  # non-finite images: only the flag matters (the reference raises)
    assert np.array_equal(d1["flags"], d0["flags"])
    for f in ("k", "k1", "k2", "nnz"):
        assert np.array_equal(d1[f][ok], d0[f][ok]), f
    for f in ("a_max", "p_tau"):
        assert np.array_equal(d1[f][ok], d0[f][ok]), f
    a, b = y1.cpu().numpy()[ok], y0.cpu().numpy()[ok]
    same = (a == b) | (np.isnan(a) & np.isnan(b))
    assert same.all(), f"{(~same).sum()} points differ"
    return y1, k1, r1


@pytest.mark.parametrize("fmt,bsz", [("e4m3", 32), ("e4m3", 16), ("e4m3", 64), ("e5m2", 32),
                                     ("e2m3", 16), ("e3m2", 64), ("e2m1", 32)])
def test_fused_small_image_matches_line_passes(mx, torch, fmt, bsz):
    """C4 phantoms (5% noise), 300 images (every CTA walks several): the fused
    kernel equals prescale statistics + four line passes bit for bit, forward
    and round trip, with identical statistics rows."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    x = ellipse_kspace_batch(300, 128, seed=77, noise=0.05)
    for rt in (False, True):
        _fused_vs_unfused(mx, torch, x, fmt, bsz, rt)


def test_fused_small_image_vs_oracle_and_edge_cases(mx, torch):
    """The fused kernel on a batch mixing phantoms with the cases its fast
    paths hand over: extreme magnitudes (exact replay of the image), values
    near 2^-60 / beyond 2^60 and skewed distributions (exact in-kernel
    statistics), all-zero and constant images, ties, a non-finite image (flag
    0), checked against the unfused path and, for the finite ones, the oracle."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    rng = np.random.default_rng(9)
    x = ellipse_kspace_batch(24, 128, seed=300, noise=0.05)
    x[1] *= np.float32(1e-30)                       # tiny: replay and statistics fallback
    x[2] *= np.float32(1e25)                        # huge keys
    x[3] = 0                                        # all zero: nnz = 0, k from EPS
    x[4] = np.complex64(3.0 + 4.0j)                 # constant: every magnitude ties
    x[5, :, :64] = 0                                # half zeros
    x[6] = (rng.standard_normal((128, 128)) * 10.0 ** rng.uniform(-20, 20, (128, 128))).astype(np.complex64)
    x[7, ::2] *= np.float32(2.0**-70)               # bimodal: half the points far below the rest
    x[8] = np.float32(2.0**-140)                    # subnormal FP32 input
    x[9, 5, 7] = np.complex64(complex(np.inf, 0))   # non-finite
    x[10, 0, 0] = np.complex64(3e38)                # one huge peak
    for rt in (False, True):
        y, k, res = _fused_vs_unfused(mx, torch, x, "e4m3", 32, rt)
        d = mx.prescale.decode_results(res)
        assert d["flags"][9] & 1 and not (d["flags"][[0, 1, 2, 3, 4, 5, 6, 7, 8, 10]] & 1).any()
        op = O.make_plan(128, O.E4M3, 32)
        yh = y.cpu().numpy()
        for i in (0, 1, 2, 3, 4, 5, 6, 7, 8, 10):
            out_o, _, k_o = O.pipeline(x[i], op, rt)
            assert int(k[i]) == k_o, i
            assert np.array_equal(yh[i].astype(np.complex128), out_o[0]), i


def test_fused_pipeline_host_and_graph(mx, torch):
    """pipeline_host (graph-captured H2D / fused kernel / D2H slices) on C4
    images equals pipeline_device."""
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    x = ellipse_kspace_batch(64, 128, seed=12, noise=0.05)
    p = mx.make_plan(128, mx.ModeSpec.mx(mx.E4M3, 32))
    cfg = mx.PrescaleConfig()
    h = torch.from_numpy(x).pin_memory()
    out = torch.empty_like(h).pin_memory()
    for _ in range(2):
        mx.pipeline_host(h, p, cfg, True, out_host=out)
    y, _, _ = mx.pipeline_device(torch.from_numpy(x).cuda(), p, cfg, True)
    assert torch.equal(out, y.cpu())


@pytest.mark.parametrize("mode", ["forward", "inverse", "roundtrip"])
def test_fused_fft2_modes_inplace_kgroups(mx, torch, mode):
    """mxfft_fft2 at n = 128 (the fused image kernel, given k) equals the four
    line passes for every mode, out of place and in place, with per-stack k
    (k_group = 2) and without k."""
    from paper_2512_04317_b200 import _native
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    x = torch.from_numpy(ellipse_kspace_batch(200, 128, seed=5, noise=0.05) * np.float32(2.0**-10)).cuda()
    k = torch.tensor(np.random.default_rng(1).integers(-6, 7, 100), dtype=torch.int32, device="cuda")
    p = mx.make_plan(128, mx.ModeSpec.mx(mx.E5M2, 16))
    L = _native.lib()
    for kk, g in ((None, 1), (k, 2)):
        L.mxfft_fused_image(0)
        try:
            want = mx.fft2_device(x, p, mode, k=kk, k_group=g)
            torch.cuda.synchronize()
            L.mxfft_fused_image(1)
            got = mx.fft2_device(x, p, mode, k=kk, k_group=g)
            assert torch.equal(got, want), (mode, g)
            y = x.clone()
            mx.fft2_device(y, p, mode, k=kk, k_group=g, out=y)
            assert torch.equal(y, want), ("in place", mode, g)
        finally:
            L.mxfft_fused_image(-1)
        auto = mx.fft2_device(x, p, mode, k=kk, k_group=g)  # the automatic choice
        assert torch.equal(auto, want), ("auto", mode, g)


def test_count_range_flush_stress_deterministic(mx, torch):
    """The global statistics' streaming pass (k_ps_count_range) with a bracket
    wide enough that every CTA flushes its shared candidate buffer many times
    (the path of the round-1 shared-memory race): 30 runs give the same
    counts and the same candidate multiset as numpy.  compute-sanitizer is
    closed on this GPU pool, so determinism under stress stands in for a
    racecheck log."""
    from paper_2512_04317_b200 import distributed as D
    from tests_cpu_keys import keys_np

    rng = np.random.default_rng(17)
    n = 1 << 21
    z = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    z[rng.random(n) < 0.1] = 0
    k = keys_np(z)
    k64 = z.real.astype(np.float64) ** 2 + z.imag.astype(np.float64) ** 2

    def clear(t):  # a threshold no key lies within 1e-5 of (so FP32 key rounding cannot matter)
        t = np.float32(t)
        while (np.abs(k64 - float(t)) <= 1e-5 * float(t)).any():
            t = np.float32(t * np.float32(1.0001))
        return t

    lo, hi = clear(0.05), clear(3.0)
    top = clear(np.sort(k64[z != 0])[-50] * 1.00002)
    want_c = np.sort_complex(z[(k >= lo) & (k <= hi) & np.isfinite(k)])
    want_t = np.sort_complex(z[(k >= top) & np.isfinite(k)])
    zd = torch.from_numpy(z).cuda()
    ops = D.CudaOps()
    first = None
    for _ in range(30):
        counts, cand, topv = ops.count_range(zd, float(lo), float(hi), float(top), n, n)
        got = (counts, np.sort_complex(cand.cpu().numpy()), np.sort_complex(topv.cpu().numpy()))
        if first is None:
            first = got
            nnz = int((z != 0).sum())
            below = int(((k < lo) & np.isfinite(k)).sum())
            assert counts[:4] == (nnz, below, len(want_c), len(want_t)) and counts[4] == 0, counts
            assert np.array_equal(got[1], want_c) and np.array_equal(got[2], want_t)
        else:
            assert got[0] == first[0] and np.array_equal(got[1], first[1]) and np.array_equal(got[2], first[2])


def test_butterfly_mx_kernel_reference_kats(mx, torch):
    """butterfly_mx / _mx_multiply_batch run as the mxfft_mx_multiply_f64 kernel;
    the reference's own known answers (tests/test_fftcore.py:109-162): unit
    twiddle with u = 0 gives decode(encode(v)), v = 0 gives u, a wide format
    converges to the exact product, renormalization keeps the bound, and the
    batched multiply equals the single-block butterfly bit for bit; plus the
    stage products of the reference capture (tests/golden/stages.npz)."""
    rng = np.random.default_rng(20240817)
    E4M3 = mx.E4M3
    v = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    y0, y1 = mx.butterfly_mx(np.zeros(4, complex), v, np.ones(4, complex), E4M3)
    inter = np.empty(8)
    inter[0::2], inter[1::2] = v.real, v.imag
    want = mx.decode_block_mx(mx.encode_block_mx(inter, E4M3)).astype(np.complex64)
    assert np.array_equal(y0, want) and np.array_equal(y1, -y0)
    u = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    y0, y1 = mx.butterfly_mx(u, np.zeros(4, complex), np.exp(-2j * np.pi * np.arange(4) / 8), E4M3)
    assert np.array_equal(y0, u.astype(np.complex64)) and np.array_equal(y1, u.astype(np.complex64))
    WIDE = mx.MinifloatFormat("wide", 8, 23, "ieee")
    u = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    v = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    w = np.exp(-2j * np.pi * rng.uniform(0, 1, 16))
    y0, y1 = mx.butterfly_mx(u, v, w, WIDE)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel(y0, u + w * v) <= 1e-6 and rel(y1, u - w * v) <= 1e-6
    m = E4M3.max_finite
    vv, ww = np.array([m + 0j, m + 0j]), np.array([m + 0j, -m + 0j])
    y0, y1 = mx.butterfly_mx(np.zeros(2, complex), vv, ww, E4M3)
    assert np.all(np.isfinite(y0)) and np.all(np.isfinite(y1))
    exact = ww * vv
    assert np.all(np.abs(y0 - exact) <= 2.0 ** np.floor(np.log2(np.abs(exact))) * 2.0**-E4M3.mantissa_bits)
    for _ in range(20):
        cpb = int(rng.choice([1, 4, 16]))
        u = rng.standard_normal(cpb) + 1j * rng.standard_normal(cpb)
        v = rng.standard_normal(cpb) + 1j * rng.standard_normal(cpb)
        w = np.exp(-2j * np.pi * rng.uniform(0, 1, cpb))
        w_enc = mx.fftcore._encode_blocks_batch(w.real[None], w.imag[None], cpb, E4M3)
        wv = mx.fftcore._mx_multiply_batch(v.real[None], v.imag[None], w_enc, E4M3, cpb)[0]
        y0, y1 = mx.butterfly_mx(u, v, w, E4M3)
        u32 = u.astype(np.complex64)
        assert np.array_equal(y0, u32 + wv.astype(np.complex64))
        assert np.array_equal(y1, u32 - wv.astype(np.complex64))
    # the reference's per-stage products (stage capture of _fft_batch, golden)
    g = golden("stages")
    for ci, case in enumerate(g["cases"]):
        name, bsz, n = str(case).split(":")
        bsz, n = int(bsz), int(n)
        fmt = mx.get_mx_format(name)
        p = mx.make_plan(n, mx.ModeSpec.mx(fmt, bsz))
        cpb = min(bsz // 2, n // 2)
        codes_r, codes_i, scales = p.mx_twiddles[n.bit_length() - 2]  # the last stage: half = n/2
        outs = g[f"c{ci}_forward_out"]  # (stages, batch, n) reference stage outputs
        st = n.bit_length() - 1
        prev = outs[st - 2].astype(np.complex128)  # input of the last stage
        half = n // 2
        vv = prev[:, half:]
        wv = mx.fftcore._mx_multiply_batch(vv.real, vv.imag, (codes_r, codes_i, scales), fmt, cpb)
        u32 = prev[:, :half].astype(np.complex64)
        got = np.concatenate([u32 + wv.astype(np.complex64), u32 - wv.astype(np.complex64)], axis=1)
        assert np.array_equal(got, outs[st - 1]), case


@pytest.mark.parametrize("n,R", [(1024, 128), (1024, 512), (16384, 2048), (16384, 8192)])
def test_rows_seg_reads_alltoall_layout(mx, torch, n, R):
    """mxfft_fft_rows_seg on an all-to-all receive buffer (G, R, R) equals the
    row pass on the permuted (materialised) rows, bit for bit, with the fused
    power-of-two scalings."""
    from paper_2512_04317_b200 import distributed as D

    G = n // R
    g = torch.Generator(device="cuda")
    g.manual_seed(n + R)
    recv = torch.complex(torch.randn((G, R, R), generator=g, device="cuda"),
                         torch.randn((G, R, R), generator=g, device="cuda")) * 2.0**-3
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    ops = D.CudaOps()
    for inv, ei, eo in ((False, 0, 0), (True, 3, -5)):
        got = ops.rows_seg(recv, p, inv, exp_in=ei, exp_out=eo)
        want = ops.rows(recv.permute(1, 0, 2).reshape(R, n).contiguous(), p, inv, exp_in=ei, exp_out=eo)
        assert torch.equal(got, want), (n, R, inv)


@pytest.mark.parametrize("G", [2, 4])
def test_slab_restore_false_is_transposed_result(mx, torch, G):
    """fft2_slab(restore=False) -- three all-to-alls per round trip, passes read
    the receive buffers directly -- leaves rank r with rows r R .. of the
    transposed result (the column slabs of A)."""
    from paper_2512_04317_b200 import distributed as D
    from paper_2512_04317_b200.workloads import ellipse_kspace

    n = 512
    x = ellipse_kspace(n, 31, noise=0.01)
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    want = mx.fft2_device(torch.from_numpy(x[None].copy()).cuda(), p, "roundtrip", k=None)[0].cpu().numpy()
    shared = {"world": G, "bar": threading.Barrier(G), "box": [None] * G}
    out = [None] * G
    errs = []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                r0, r1 = D.shard_range(n, r, G)
                xs = torch.from_numpy(x[r0:r1].copy()).cuda()
                y = D.fft2_slab(xs, p, "roundtrip", comm=ThreadComm(shared, r), restore=False)
                torch.cuda.current_stream().synchronize()
                out[r] = y.cpu().numpy()
        except BaseException as e:
            errs.append(e)
            shared["bar"].abort()

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(G)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs[0]
    assert np.array_equal(np.concatenate(out), want.T)


@pytest.mark.parametrize("fmt,bsz", [("e4m3", 32), ("e5m2", 16)])
def test_split_last_stage_fft2_16384(mx, torch, fmt, bsz):
    """n = 16384 passes as stages 0-12 on the decimated half rows (the
    8192-point line kernel) + the last stage fused into the transposed store
    equal the 14-stage row kernel + tiled transpose, bit for bit, for every
    mode with k; rows scaled to extreme magnitudes exercise the exact replay
    of the half rows and the inline exact path of the fused last stage."""
    from paper_2512_04317_b200 import _native
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    n = 16384
    x = ellipse_kspace_device(n, 9, noise=0.01) * (2.0**-12)
    x[:3] *= 2.0**-110   # tiny rows: out of the fast range (subnormal block maxima)
    x[5] *= 2.0**40      # large row (intermediates stay finite: the reference raises on non-finite ones)
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    L = _native.lib()
    k = torch.tensor([-3], dtype=torch.int32, device="cuda")
    for mode in ("forward", "inverse", "roundtrip"):
        L.mxfft_split_last_stage(0)
        try:
            want = mx.fft2_device(x[None], p, mode, k=k)
            torch.cuda.synchronize()
        finally:
            L.mxfft_split_last_stage(1)
        got = mx.fft2_device(x[None], p, mode, k=k)
        same = (got == want) | (torch.isnan(got) & torch.isnan(want))
        assert bool(same.all()), (mode, int((~same).sum()))
        del got, want
        torch.cuda.empty_cache()
