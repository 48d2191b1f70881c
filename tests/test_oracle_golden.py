"""Pin the CPU oracle (oracle/mxfft_oracle.c) to outputs of the reference itself.

The fixtures were produced by tests/golden/make_golden.py, which imports the
unmodified reference package; every comparison here is bit-exact (value
equality -- the reference turns an imaginary -0 code into +0, fftcore.py:182)."""

import numpy as np
import pytest

import oracle as O
from conftest import golden

FMTS = O.ALL_MX


def test_quantize_matches_reference():
    g = golden("quantize")
    for name in list(FMTS) + ["fp16"]:
        f = FMTS.get(name, O.FP16)
        got = O.quantize_array(g[f"{name}_x"], f)
        assert np.array_equal(got, g[f"{name}_q"]), name


def test_format_constants():
    # reference tests/test_minifloat.py:28-51 (+ E2M1)
    assert O.E4M3.info() == dict(emin=-6, emax=8, max_finite=448.0, min_subnormal=2.0**-9)
    assert O.E5M2.info()["max_finite"] == 57344.0 and O.E5M2.info()["emax"] == 15
    assert O.E2M3.info()["max_finite"] == 7.5
    assert O.E3M2.info()["max_finite"] == 28.0
    assert O.E2M1.info() == dict(emin=0, emax=2, max_finite=6.0, min_subnormal=0.5)
    assert O.FP16.info()["max_finite"] == 65504.0


def test_mx_block_kat():
    # reference tests/test_mxblock.py:38-45: [1, .5, -.25, 0] -> scale 2^-8, codes [256,128,-64,0]
    cr, ci, sc = O.encode_blocks([[1.0, -0.25]], [[0.5, 0.0]], 2, O.E4M3)
    assert sc[0, 0] == 2.0**-8
    assert np.array_equal(cr.ravel(), [256.0, -64.0]) and np.array_equal(ci.ravel(), [128.0, 0.0])


def test_twiddles_match_reference():
    g = golden("twiddles")
    for name, f in FMTS.items():
        for bsz in (2, 32):
            for n in (8, 256):
                p = O.make_plan(n, f, bsz)
                key = f"{name}_{bsz}_{n}"
                assert np.array_equal(O.ref_twiddles(n), g[key + "_ref"])
                assert np.array_equal(p.wcr, g[key + "_cr"].reshape(p.wcr.shape)), key
                assert np.array_equal(p.wci, g[key + "_ci"].reshape(p.wci.shape)), key
                assert np.array_equal(p.ws, g[key + "_s"].reshape(p.ws.shape)), key


def test_batch_fft_matches_reference():
    g = golden("batch")
    for ci, case in enumerate(g["cases"]):
        name, bsz, n = str(case).split(":")
        p = O.make_plan(int(n), FMTS[name], int(bsz))
        x = g[f"c{ci}_x"]
        assert np.array_equal(O.fft_batch(x, p, False), g[f"c{ci}_fwd"]), case
        assert np.array_equal(O.fft_batch(x, p, True), g[f"c{ci}_inv"]), case


def test_stage_capture_matches_reference():
    """Per-stage v-block exponents and codes, product exponents/codes/shifts and
    stage outputs, captured from the reference by wrapping its functions."""
    g = golden("stages")
    for ci, case in enumerate(g["cases"]):
        name, bsz, n = str(case).split(":")
        p = O.make_plan(int(n), FMTS[name], int(bsz))
        x = g[f"c{ci}_x"]
        for direction in ("forward", "inverse"):
            y, cap = O.fft_batch(x, p, direction == "inverse", dump=True)
            pre = f"c{ci}_{direction}_"
            assert np.array_equal(y, g[pre + "y"])
            assert np.array_equal(cap["v_exp"], g[pre + "v_exp"]), case
            assert np.array_equal(cap["v_codes"], g[pre + "v_codes"]), case
            assert np.array_equal(cap["p_codes"], g[pre + "p_codes"]), case
            assert np.array_equal(cap["p_exp"], g[pre + "p_exp"]), case
            assert np.array_equal(cap["p_shift"], g[pre + "p_shift"]), case
            assert np.array_equal(cap["stage_out"], g[pre + "out"]), case


def test_fft2_matches_reference():
    g = golden("fft2")
    for ci, case in enumerate(g["cases"]):
        name, bsz, n = str(case).split(":")
        p = O.make_plan(int(n), FMTS[name], int(bsz))
        x = g[f"c{ci}_x"]
        assert np.array_equal(O.fft2(x, p, False), g[f"c{ci}_fwd"]), case
        assert np.array_equal(O.fft2(x, p, True), g[f"c{ci}_inv"]), case


def test_prescale_matches_reference():
    g = golden("prescale")
    for i in range(int(g["count"])):
        r = O.compute_prescale(g[f"x{i}"])
        assert [r.k, r.k1, r.k2] == list(g["k"][i]), i
        assert r.a_max == g[f"am{i}"][0] and r.p_tau == g[f"am{i}"][1], i


def test_cabs_matches_numpy():
    g = golden("prescale")
    assert np.array_equal(O.cabs(g["abs_x"]), g["abs_y"])


def test_pipelines_match_reference():
    g = golden("pipelines")
    for ci, case in enumerate(g["cases"]):
        name, bsz, n = str(case).split(":")
        p = O.make_plan(int(n), FMTS[name], int(bsz))
        x = g[f"c{ci}_x"]
        _, rss_f, k = O.pipeline(x, p, False)
        _, rss_r, _ = O.pipeline(x, p, True)
        assert k == int(g[f"c{ci}_k"])
        assert np.array_equal(rss_f, g[f"c{ci}_fwd_rss"]), case
        assert np.array_equal(rss_r, g[f"c{ci}_rt_rss"]), case


def test_prescale_kats():
    # reference tests/test_prescale.py:43-75 and tests/test_acceptance.py:225-236
    r = O.compute_prescale(np.array([1.0, 0.5, 0.25], dtype=complex))
    assert (r.k1, r.k, r.a_max) == (0, 0, 1.0)
    assert O.compute_prescale(np.array([0.25, 0.1], dtype=complex)).k == 2
    z = O.compute_prescale(np.zeros((4, 4), dtype=complex))
    assert z.a_max == 0.0 and z.p_tau == 0.0 and z.k == 40
    assert (O.compute_prescale(np.full((4, 4), 8.0 + 0j)).k1, O.compute_prescale(np.full((4, 4), 8.0 + 0j)).k) == (-3, -3)
    t = np.full((16, 16), 2.0**-30, dtype=complex)
    t[0, 0] = 1.0
    r = O.compute_prescale(t)
    assert (r.k1, r.k2, r.k) == (0, 10, 10)
    c = O.compute_prescale(np.full((4, 4), 2.0**-60))
    assert (c.k1, c.k) == (60, 40)


# ---------------------------------------------------------------------------
# the BASELINE shapes (C3 512^2 x 9 format/block pairs, C4 128^2 5% noise,
# C5 16384-point rows), pinned to digests of the reference's own outputs
# ---------------------------------------------------------------------------
from conftest import bigshape_cases, bigshape_image, digest  # noqa: E402


@pytest.mark.parametrize("case", bigshape_cases(), ids=lambda c: c[0])
def test_oracle_baseline_shapes_match_reference(case):
    key, tag, fmt, bsz, i = case
    g = golden("bigshapes")
    x = bigshape_image(tag, i)
    assert digest(x) == str(g[key + "_x"]), "input generator differs from the fixture's"
    p = O.make_plan(x.shape[0], FMTS[fmt], bsz)
    pr = O.compute_prescale(x)
    assert [pr.k, pr.k1, pr.k2] == g[key + "_k"].tolist()
    assert [pr.a_max, pr.p_tau] == g[key + "_stats"].tolist()
    out_f, rss_f, kf = O.pipeline(x, p, False)
    out_r, rss_r, kr = O.pipeline(x, p, True)
    assert kf == kr == pr.k
    assert digest(out_f[0]) == str(g[key + "_fwd"])
    assert digest(out_r[0]) == str(g[key + "_rt"])
    assert digest(rss_f) == str(g[key + "_fwd_rss"])
    assert digest(rss_r) == str(g[key + "_rt_rss"])


def test_oracle_c5_rows_match_reference():
    g = golden("bigshapes")
    rows = g["c5_rows_x"]
    for fmt, bsz in (("e4m3", 32), ("e2m1", 64)):
        p = O.make_plan(16384, FMTS[fmt], bsz)
        for inv, d in ((False, "forward"), (True, "inverse")):
            assert digest(O.fft_batch(rows, p, inv)) == str(g[f"c5_{fmt}_b{bsz}_{d}"]), (fmt, d)
