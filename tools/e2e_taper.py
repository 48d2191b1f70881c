"""pipeline_host (C2 round trip): slice-weight schemes x slice counts, graph replay.
usage: python tools/e2e_taper.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import mri  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

B, n = 256, 256
hx = torch.from_numpy(ellipse_kspace_batch(B, n, seed=0)).pin_memory()
hy = torch.empty_like(hx).pin_memory()
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
orig = mri.host_slices


def weights_slices(w):
    def f(nstack, chunks):
        ww = w(chunks)
        tot = float(sum(ww))
        sizes = [max(1, int(nstack * x / tot)) for x in ww]
        sizes[len(sizes) // 2] += nstack - sum(sizes)
        return sizes
    return f


schemes = {
    "current": orig,
    "taper": weights_slices(lambda c: [min(4, 2 ** i, 2 ** (c - 1 - i)) for i in range(c)]),
    "taper8": weights_slices(lambda c: [min(8, 2 ** i, 2 ** (c - 1 - i)) for i in range(c)]),
    "flat": weights_slices(lambda c: [1] * c),
}


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ref = None
for name, fn in schemes.items():
    mri.host_slices = fn
    for ch in (8, 10, 12, 16, 24):
        mri._HOST_GRAPHS.clear()
        ms = t(lambda: mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=ch, graph=True))
        if ref is None:
            ref = hy.clone()
        same = torch.equal(torch.view_as_real(ref), torch.view_as_real(hy))
        print(f"{name:8s} chunks={ch:3d} {ms:.3f} ms  {B * n * n / ms / 1e6:.2f} Gpoints/s  same={same}  "
              f"sizes={fn(B, ch)}", flush=True)
