"""pipeline_host (C2 round trip) over slice counts, eager and graph-replayed.
usage: python tools/e2e_sweep.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

B, n = 256, 256
hx = torch.from_numpy(ellipse_kspace_batch(B, n, seed=0)).pin_memory()
hy = torch.empty_like(hx).pin_memory()
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()


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
for graph in (False, True):
    for ch in (8, 16, 24, 32, 48, 64):
        ms = t(lambda: mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=ch, graph=graph))
        same = True
        if ref is None:
            ref = hy.clone()
        else:
            same = torch.equal(torch.view_as_real(ref), torch.view_as_real(hy))
        print(f"graph={graph} chunks={ch}: {ms:.3f} ms  {B * n * n / ms / 1e6:.2f} Gpoints/s  same={same}")
