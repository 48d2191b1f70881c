"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only under the alias ``mxfft_ref``
(leaving the name ``mxfft`` free), runs it on seeded inputs, and writes small
.npz files.  Per-stage MX exponents/codes are captured by wrapping the
reference's own module-level functions (``_encode_blocks_batch``,
``quantize_array``, ``_mx_multiply_batch``) -- the reference source is not
modified or copied.  The GPU box never runs this script; the fixtures travel
with the repo and tests/test_oracle_golden.py pins the C oracle to them.
"""

from __future__ import annotations

import copy
import importlib.util
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src/mxfft"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(OUT, "..", ".."))
from paper_2512_04317_b200.workloads import ellipse_kspace  # noqa: E402  (host-only generator)


def load_ref():
    spec = importlib.util.spec_from_file_location(
        "mxfft_ref", os.path.join(REF, "__init__.py"), submodule_search_locations=[REF]
    )
    mod = importlib.util.module_from_spec(spec)
    sys.modules["mxfft_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


R = load_ref()
E2M1 = R.MinifloatFormat("e2m1", 2, 1, "finite")
FMTS = {"e4m3": R.E4M3, "e5m2": R.E5M2, "e2m3": R.E2M3, "e3m2": R.E3M2, "e2m1": E2M1}


def quantize_fixture(rng):
    out = {}
    for name, f in list(FMTS.items()) + [("fp16", R.FP16)]:
        grid = R.enumerate_values(f)
        mids = (grid[:-1] + grid[1:]) / 2.0
        hi = R.quantize_scalar(1e300, f)
        vals = np.concatenate([
            grid, mids, np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf),
            rng.uniform(-2 * hi, 2 * hi, 2000),
            rng.standard_normal(2000) * 2.0 ** rng.uniform(-30, 20, 2000),
            [0.0, -0.0, 1e-300, -1e-300, 1e30, -1e30, f.min_subnormal / 2, f.min_subnormal / 4],
        ])
        out[f"{name}_x"] = vals
        out[f"{name}_q"] = R.quantize_array(vals, f)
    return out


def batch_fixture(rng):
    out = {}
    cases = []
    for name in FMTS:
        for bsz in (2, 8, 32, 64):
            for n in (8, 64, 256):
                cases.append((name, bsz, n))
    for ci, (name, bsz, n) in enumerate(cases):
        x = (rng.standard_normal((2, n)) + 1j * rng.standard_normal((2, n))) * 10.0 ** rng.uniform(-3, 3)
        plan = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
        out[f"c{ci}_x"] = x
        out[f"c{ci}_fwd"] = R.fftcore._fft_batch(x, plan, "forward")
        out[f"c{ci}_inv"] = R.fftcore._fft_batch(x, plan, "inverse")
    out["cases"] = np.array([f"{a}:{b}:{c}" for a, b, c in cases])
    return out


def capture_stages(x, plan, direction):
    """Run the reference batch transform and record, per stage, the v-block scale
    exponents and codes, product exponents/codes/shifts, and stage output."""
    fc = R.fftcore
    rec = {"v_exp": [], "v_codes": [], "p_exp": [], "p_codes": [], "p_shift": [], "out": []}
    orig_mul, orig_enc, orig_q = fc._mx_multiply_batch, fc._encode_blocks_batch, fc.quantize_array
    state = {}

    def enc(vr, vi, cpb, fmt):
        r = orig_enc(vr, vi, cpb, fmt)
        if state.get("in_mul"):
            state["venc"] = r
        return r

    def q(values, fmt):
        r = orig_q(values, fmt)
        if state.get("in_mul") and "venc" in state:
            state.setdefault("pq", []).append(r)
        return r

    def mul(vr, vi, w_enc, fmt, cpb):
        state.clear()
        state["in_mul"] = True
        wv = orig_mul(vr, vi, w_enc, fmt, cpb)
        state["in_mul"] = False
        cvr, cvi, sv = state["venc"]
        c_r, c_i = state["pq"][-2], state["pq"][-1]
        b = vr.shape[0]
        rec["v_exp"].append(np.round(np.log2(sv)).astype(np.int32))
        rec["v_codes"].append(np.stack([cvr.reshape(b, -1), cvi.reshape(b, -1)], -1))
        rec["p_codes"].append(np.stack([c_r.reshape(b, -1), c_i.reshape(b, -1)], -1))
        ws = w_enc[2]
        s_out = np.empty(c_r.shape[:2])
        wvb = wv.reshape(c_r.shape)
        for i in range(c_r.shape[0]):
            for k in range(c_r.shape[1]):
                cc = np.concatenate([c_r[i, k], c_i[i, k]])
                ww = np.concatenate([wvb[i, k].real, wvb[i, k].imag])
                nz = cc != 0
                s_out[i, k] = (ww[nz][0] / cc[nz][0]) if nz.any() else ws[0, k] * sv[i, k]
        base = np.log2(ws * sv)
        pe = np.round(np.log2(s_out)).astype(np.int32)
        rec["p_exp"].append(pe)
        rec["p_shift"].append((pe - np.round(base)).astype(np.int32))
        return wv

    fc._mx_multiply_batch, fc._encode_blocks_batch, fc.quantize_array = mul, enc, q
    try:
        y = fc._fft_batch(x, plan, direction)
    finally:
        fc._mx_multiply_batch, fc._encode_blocks_batch, fc.quantize_array = orig_mul, orig_enc, orig_q
    # stage outputs: a shallow copy of the plan whose stage count is truncated
    # (the plan object is an ordinary instance; the reference code is untouched)
    for s in range(plan.stages):
        p2 = copy.copy(plan)
        p2.stages = s + 1
        rec["out"].append(fc._fft_batch(x, p2, direction))
    return {k: np.stack(v) for k, v in rec.items() if v}, y


def stage_fixture(rng):
    out = {}
    cases = [("e4m3", 32, 256), ("e5m2", 16, 64), ("e2m1", 8, 32), ("e3m2", 64, 128), ("e2m3", 2, 16)]
    for ci, (name, bsz, n) in enumerate(cases):
        img = ellipse_kspace(n, seed=100 + ci, noise=0.01)
        x = img[: 4].astype(np.complex128) * 2.0 ** -14  # four k-space rows, prescale-like range
        plan = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
        for direction in ("forward", "inverse"):
            rec, y = capture_stages(x, plan, direction)
            for k, v in rec.items():
                out[f"c{ci}_{direction}_{k}"] = v
            out[f"c{ci}_{direction}_y"] = y
        out[f"c{ci}_x"] = x
    out["cases"] = np.array([f"{a}:{b}:{c}" for a, b, c in cases])
    return out


def fft2_fixture(rng):
    out = {}
    cases = [(f, 32, 32) for f in FMTS] + [("e4m3", 16, 64), ("e5m2", 64, 64), ("e4m3", 32, 128)]
    for ci, (name, bsz, n) in enumerate(cases):
        x = ellipse_kspace(n, seed=200 + ci, noise=0.01).astype(np.complex128) * 2.0 ** -10
        plan = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
        out[f"c{ci}_x"] = x
        out[f"c{ci}_fwd"] = R.fft_2d(x, plan, "forward")
        out[f"c{ci}_inv"] = R.fft_2d(x, plan, "inverse")
    out["cases"] = np.array([f"{a}:{b}:{c}" for a, b, c in cases])
    return out


def modes_fixture(rng):
    """The non-MX ModeSpec kinds: FP16 positive control and FP64 reference,
    1-D batches (complex128 and complex64 inputs) and 2-D transforms."""
    out = {}
    cases = [("fp16", 8), ("fp16", 64), ("fp16", 256), ("reference", 8), ("reference", 64), ("reference", 1024)]
    for ci, (kind, n) in enumerate(cases):
        plan = R.make_plan(n, R.ModeSpec.from_name(kind))
        x = (rng.standard_normal((3, n)) + 1j * rng.standard_normal((3, n))) * 10.0 ** rng.uniform(-2, 2, (3, 1))
        x32 = x.astype(np.complex64)
        out[f"c{ci}_x"] = x
        out[f"c{ci}_x32"] = x32
        for d in ("forward", "inverse"):
            out[f"c{ci}_{d}"] = R.fftcore._fft_batch(x, plan, d)
            out[f"c{ci}_{d}32"] = R.fftcore._fft_batch(x32, plan, d)
        if n <= 256:
            img = ellipse_kspace(n, seed=300 + ci, noise=0.01).astype(np.complex128) * 2.0 ** -12
            out[f"c{ci}_img"] = img
            out[f"c{ci}_fft2"] = R.fft_2d(img, plan, "forward")
            out[f"c{ci}_ifft2"] = R.fft_2d(img, plan, "inverse")
    out["cases"] = np.array([f"{a}:{b}" for a, b in cases])
    return out


def metrics_fixture(rng):
    """Reference PSNR / NMSE / SSIM (metrics.py) on seeded magnitude-image pairs."""
    out = {}
    cases = [(64, 0.01), (128, 0.1), (33, 0.5), (256, 1e-4)]
    for ci, (n, eps) in enumerate(cases):
        ref = np.abs(ellipse_kspace(n, seed=400 + ci, noise=0.0)).astype(np.float64) ** 0.5
        test = ref + eps * ref.max() * rng.standard_normal(ref.shape)
        out[f"c{ci}_ref"] = ref
        out[f"c{ci}_test"] = test
        out[f"c{ci}_vals"] = np.array([R.psnr(ref, test), R.nmse(ref, test), R.ssim(ref, test)])
    out["cases"] = np.array([f"{a}:{b}" for a, b in cases])
    return out


def phantoms_fixture(rng):
    """gen_phantom / coil_sensitivities outputs and MXCG file bytes."""
    import tempfile

    out = {}
    cases = [(32, 2, 5, "blobs", 0.1, 1e-4), (64, 1, 6, "bars", 0.0, 1e-4), (16, 3, 7, "blobs", 0.0, 0.0)]
    for ci, (n, coils, seed, kind, tail, noise) in enumerate(cases):
        img, ksp = R.gen_phantom(n, coils, seed, kind=kind, tail=tail, noise=noise)
        out[f"c{ci}_img"] = img.data
        out[f"c{ci}_ksp"] = ksp.data
        with tempfile.NamedTemporaryFile(suffix=".mxcg") as f:
            R.write_grid(ksp, f.name)
            out[f"c{ci}_mxcg"] = np.frombuffer(open(f.name, "rb").read(), dtype=np.uint8)
    out["sens"] = R.coil_sensitivities(16, 4, 3)
    out["cases"] = np.array([f"{a}:{b}:{c}:{d}:{e}:{f}" for a, b, c, d, e, f in cases])
    return out


def multicoil_fixture(rng):
    """forward_pipeline / roundtrip_pipeline on multi-coil phantom stacks (one
    global prescale per stack, RSS over coils)."""
    out = {}
    cases = [("e4m3", 32, 64, 4, "blobs"), ("e5m2", 16, 32, 3, "bars"), ("e2m1", 32, 64, 2, "blobs")]
    cfg = R.PrescaleConfig()
    for ci, (name, bsz, n, coils, kind) in enumerate(cases):
        img, ksp = R.gen_phantom(n, coils, 50 + ci, kind=kind, tail=0.05)
        plan = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
        out[f"c{ci}_ksp"] = ksp.data
        out[f"c{ci}_img"] = img.data
        out[f"c{ci}_fwd"] = R.forward_pipeline(ksp, plan, cfg).pixels
        out[f"c{ci}_rt"] = R.roundtrip_pipeline(img, plan, cfg).pixels
    out["cases"] = np.array([f"{a}:{b}:{c}:{d}:{e}" for a, b, c, d, e in cases])
    return out


def prescale_fixture(rng):
    cfg = R.PrescaleConfig()
    inputs = []
    inputs.append(np.array([1.0, 0.5, 0.25], dtype=complex))
    inputs.append(np.array([0.25, 0.1], dtype=complex))
    inputs.append(np.zeros(16, dtype=complex))
    t = np.ones(1000, dtype=complex)
    t[:500] = 2.0**-30
    inputs.append(t)
    inputs.append(np.array([2.0**-60], dtype=complex))
    inputs.append(np.full(16, 8.0 + 0j))
    t = np.full(256, 2.0**-30, dtype=complex)
    t[0] = 1.0
    inputs.append(t)
    for i in range(20):
        x = (rng.standard_normal(300) + 1j * rng.standard_normal(300)) * 10.0 ** rng.uniform(-12, 12)
        x[rng.random(300) < 0.2] = 0
        inputs.append(x.astype(np.complex64).astype(np.complex128))
    for i in range(4):
        inputs.append(ellipse_kspace(64, seed=300 + i, noise=0.01).reshape(-1).astype(np.complex128))
    out = {}
    res = []
    for i, x in enumerate(inputs):
        r = R.compute_prescale(x, cfg)
        out[f"x{i}"] = x
        res.append([r.k, r.k1, r.k2])
        out[f"am{i}"] = np.array([r.a_max, r.p_tau])
    out["k"] = np.array(res, dtype=np.int64)
    out["count"] = np.array(len(inputs))
    z = (rng.standard_normal(5000) + 1j * rng.standard_normal(5000)) * 10.0 ** rng.uniform(-30, 30, 5000)
    out["abs_x"] = z
    out["abs_y"] = np.abs(z)
    return out


def pipeline_fixture(rng):
    cfg = R.PrescaleConfig()
    out = {}
    cases = [("e4m3", 32, 64), ("e5m2", 32, 64), ("e3m2", 16, 32), ("e2m3", 64, 32), ("e2m1", 32, 32),
             ("e4m3", 32, 128)]
    for ci, (name, bsz, n) in enumerate(cases):
        ksp = ellipse_kspace(n, seed=400 + ci, noise=0.01).astype(np.complex128)
        plan = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
        fwd = R.forward_pipeline(R.ComplexGrid(ksp[None], "kspace"), plan, cfg)
        rt = R.roundtrip_pipeline(R.ComplexGrid(ksp[None], "image"), plan, cfg)
        out[f"c{ci}_x"] = ksp
        out[f"c{ci}_fwd_rss"] = fwd.pixels
        out[f"c{ci}_rt_rss"] = rt.pixels
        out[f"c{ci}_k"] = np.array(R.compute_prescale(ksp, cfg).k)
    out["cases"] = np.array([f"{a}:{b}:{c}" for a, b, c in cases])
    return out


def twiddle_fixture(rng):
    out = {}
    for name in FMTS:
        for bsz in (2, 32):
            for n in (8, 256):
                p = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
                out[f"{name}_{bsz}_{n}_ref"] = np.stack(p.ref_twiddles)
                out[f"{name}_{bsz}_{n}_cr"] = np.stack([t[0][0] for t in p.mx_twiddles])
                out[f"{name}_{bsz}_{n}_ci"] = np.stack([t[1][0] for t in p.mx_twiddles])
                out[f"{name}_{bsz}_{n}_s"] = np.stack([t[2][0] for t in p.mx_twiddles])
    return out


def digest(a) -> str:
    """SHA-256 of an array's values (C order; -0.0 folded into +0.0, since the
    reference compares by value).  Large reference outputs are pinned by
    digest: the fixture stays small and the comparison stays bit-exact."""
    import hashlib

    a = np.ascontiguousarray(np.asarray(a) + 0.0)
    return hashlib.sha256(a.tobytes()).hexdigest()


def bigshapes_fixture(rng):
    """The BASELINE configurations' own shapes, pinned by digests of the
    reference's outputs:
      C3: one 512^2 phantom, E3M2 / E2M3 / E2M1 x B in {16, 32, 64};
      C4: four 128^2 phantoms with 5% noise, E4M3 B=32;
      C5: two 16384-point rows, E4M3 B=32 and E2M1 B=64, forward and inverse.
    For each pipeline case: k, a_max, p_tau, the per-coil complex outputs of
    forward_pipeline / roundtrip_pipeline's body (mri.py:84-107: apply_prescale,
    fft_2d [, fft_2d inverse x 1/N^2], undo_prescale) and the RSS images the
    public pipelines return.  Inputs come from the seeded generator
    (workloads.ellipse_kspace); their digests are stored so that a different
    numpy on another host fails loudly instead of comparing other inputs."""
    rng = np.random.default_rng(5120)  # own stream: the older fixtures stay byte-identical
    cfg = R.PrescaleConfig()
    out = {}
    cases = []
    imgs = {"c3": [ellipse_kspace(512, seed=501, noise=0.01)],
            "c4": [ellipse_kspace(128, seed=601 + i, noise=0.05) for i in range(4)]}
    combos = [("c3", f, b) for f in ("e3m2", "e2m3", "e2m1") for b in (16, 32, 64)] + [("c4", "e4m3", 32)]
    for tag, name, bsz in combos:
        for ii, x64 in enumerate(imgs[tag]):
            x = x64.astype(np.complex128)
            n = x.shape[0]
            plan = R.make_plan(n, R.ModeSpec.mx(FMTS[name], bsz))
            pr = R.compute_prescale(x, cfg)
            xs = R.apply_prescale(x, pr.k)
            fwd = R.fft_2d(xs, plan, "forward")
            rt = R.fft_2d(fwd, plan, "inverse") * (1.0 / (n * n))
            key = f"{tag}_{name}_b{bsz}_i{ii}"
            cases.append(key)
            out[key + "_x"] = np.array(digest(x64))
            out[key + "_k"] = np.array([pr.k, pr.k1, pr.k2])
            out[key + "_stats"] = np.array([pr.a_max, pr.p_tau])
            out[key + "_fwd"] = np.array(digest(R.undo_prescale(fwd, pr.k)))
            out[key + "_rt"] = np.array(digest(R.undo_prescale(rt, pr.k)))
            out[key + "_fwd_rss"] = np.array(digest(
                R.forward_pipeline(R.ComplexGrid(x[None], "kspace"), plan, cfg).pixels))
            rt_rss = R.roundtrip_pipeline(R.ComplexGrid(x[None], "image"), plan, cfg).pixels
            out[key + "_rt_rss"] = np.array(digest(rt_rss))
            ref = np.abs(x)
            out[key + "_quality"] = np.array([R.psnr(ref, rt_rss), R.nmse(ref, rt_rss)])
            print(key, pr.k, flush=True)
    rows = ((rng.standard_normal((2, 16384)) + 1j * rng.standard_normal((2, 16384))) * 2.0 ** -6).astype(np.complex64)
    out["c5_rows_x"] = rows
    for name, bsz in (("e4m3", 32), ("e2m1", 64)):
        plan = R.make_plan(16384, R.ModeSpec.mx(FMTS[name], bsz))
        for d in ("forward", "inverse"):
            out[f"c5_{name}_b{bsz}_{d}"] = np.array(digest(R.fftcore._fft_batch(rows.astype(np.complex128), plan, d)))
            cases.append(f"c5_{name}_b{bsz}_{d}")
    out["cases"] = np.array(cases)
    return out


FIXTURES = [("quantize", quantize_fixture), ("batch", batch_fixture),
            ("stages", stage_fixture), ("fft2", fft2_fixture),
            ("prescale", prescale_fixture), ("pipelines", pipeline_fixture),
            ("twiddles", twiddle_fixture), ("modes", modes_fixture),
            ("metrics", metrics_fixture), ("phantoms", phantoms_fixture),
            ("multicoil", multicoil_fixture), ("bigshapes", bigshapes_fixture)]


def main():
    """Regenerate every fixture, or only those named on the command line (the
    shared rng is advanced through every fixture either way, so a partial run
    writes exactly the bytes a full run would)."""
    only = set(sys.argv[1:])
    rng = np.random.default_rng(20240817)
    for name, fn in FIXTURES:
        if only and name not in only and name == "bigshapes":
            continue
        data = fn(rng)
        if only and name not in only:
            continue
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **data)
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
