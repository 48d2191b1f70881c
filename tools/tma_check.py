"""TMA transposed store (n = 256 / 512) against the per-thread copy-out: equal
results for every format / block size / mode, then per-pass times of the C2
and C3 shapes with the knob off and on (same process, alternating)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

L = _native.lib()
ok = True
L.mxfft_fused_image(0)  # n = 128: the line passes, not the fused image kernel
for n, batch in ((128, 70), (256, 24), (512, 10)):
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=3)).cuda()
    kk = torch.arange(batch, dtype=torch.int32, device="cuda") % 7 - 3
    for fmt in ("e4m3", "e5m2", "e3m2", "e2m3", "e2m1"):
        for B in (16, 32, 64):
            plan = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), B))
            for mode in ("forward", "inverse", "roundtrip"):
                outs = []
                for on in (0, 1):
                    L.mxfft_tma_store(on)
                    y = torch.empty_like(x)
                    mx.fft2_device(x, plan, mode, k=kk, out=y)
                    torch.cuda.synchronize()
                    outs.append(y)
                same = torch.equal(torch.view_as_real(outs[0]), torch.view_as_real(outs[1]))
                ok &= same
                if not same:
                    d = (torch.view_as_real(outs[0]) != torch.view_as_real(outs[1])).any(-1)
                    print(f"MISMATCH n={n} {fmt} B={B} {mode}: {int(d.sum())} points differ, first {d.nonzero()[0].tolist()}")
print("tma store equals copy-out:", ok)


def time_case(n, batch, fmt, B, mode, reps=30):
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda() * (2.0 ** -14)
    y = torch.empty_like(x)
    plan = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), B))
    res = {0: [], 1: []}
    for rnd in range(5):
        for on in (0, 1):
            L.mxfft_tma_store(on)
            for _ in range(3):
                mx.fft2_device(x, plan, mode, out=y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                mx.fft2_device(x, plan, mode, out=y)
            e1.record()
            torch.cuda.synchronize()
            res[on].append(e0.elapsed_time(e1) / reps * 1e3 / (4 if mode == "roundtrip" else 2))
    for on in (0, 1):
        v = sorted(res[on])
        print(f"n={n} batch={batch} {fmt} B={B} {mode} tma={on}: us/pass median {v[2]:.1f} min {v[0]:.1f}")


def time_pdl(n, batch, fmt, B, reps=30):
    """round-trip pipeline (statistics + passes) with programmatic dependent launch off / on"""
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda()
    y = torch.empty_like(x)
    plan = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), B))
    cfg = mx.PrescaleConfig()
    res = {0: [], 1: []}
    outs = {}
    for rnd in range(5):
        for on in (0, 1):
            L.mxfft_pdl(on)
            for _ in range(3):
                mx.pipeline_device(x, plan, cfg, roundtrip=True, out=y)
            torch.cuda.synchronize()
            outs[on] = y.clone()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                mx.pipeline_device(x, plan, cfg, roundtrip=True, out=y)
            e1.record()
            torch.cuda.synchronize()
            res[on].append(e0.elapsed_time(e1) / reps * 1e3)
    same = torch.equal(torch.view_as_real(outs[0]), torch.view_as_real(outs[1]))
    for on in (0, 1):
        v = sorted(res[on])
        print(f"pipeline n={n} batch={batch} {fmt} B={B} pdl={on}: us/step median {v[2]:.1f} min {v[0]:.1f} same={same}")


time_case(128, 4096, "e4m3", 32, "roundtrip")
time_pdl(128, 4096, "e4m3", 32)
L.mxfft_fused_image(1)
time_pdl(256, 256, "e4m3", 32)
time_pdl(512, 64, "e3m2", 32)
time_pdl(128, 4096, "e4m3", 32)
L.mxfft_pdl(1)
time_case(256, 256, "e4m3", 32, "forward")
time_case(256, 256, "e4m3", 32, "roundtrip")
time_case(512, 64, "e3m2", 32, "forward")
time_case(512, 64, "e2m1", 16, "roundtrip")
L.mxfft_tma_store(1)
