"""How much of a pass is memory, compute, and their overlap: fft2 forward
timed with the line kernel's profiling knobs (skip loads / skip stores /
both).  usage: python tools/overlap.py [n] [batch]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda() * (2.0 ** -14)
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
y = torch.empty_like(x)
ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, batch)), dtype=torch.uint8,
                 device="cuda")
L = _native.lib()


def t(reps=30):
    f = lambda: mx.fft2_device(x, plan, "forward", out=y, workspace=ws)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3 / 2


for flags, what in ((0, "full pass"), (1, "no loads"), (2, "no stores"), (3, "compute only")):
    for lim in (-1, 0):
        L.mxfft_profile_flags(flags)
        L.mxfft_profile_stage_limit(lim)
        print(f"n={n} batch={batch} {what:13s} stages={'all' if lim < 0 else lim:>3}: {t():7.1f} us/pass")
L.mxfft_profile_flags(0)
L.mxfft_profile_stage_limit(-1)
