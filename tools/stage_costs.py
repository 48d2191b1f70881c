"""Cost of a line pass as a function of how many stages run (profiling only:
with a stage cap the output is not a transform).  usage: python tools/stage_costs.py [n] [batch]"""
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
L = _native.lib()


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


out = []
for lim in list(range(0, plan.stages + 1)):
    L.mxfft_profile_stage_limit(lim if lim < plan.stages else -1)
    out.append((lim, t(lambda: mx.fft_rows_device(x, plan, False, out=y)),
                t(lambda: mx.fftcore.fft_cols_device(x, plan, False, out=y))))
L.mxfft_profile_stage_limit(-1)
print(f"n={n} batch={batch}: stages -> rows_us / cols_us")
for lim, r, c in out:
    print(f"  {lim:2d}: {r:7.1f} {c:7.1f}")
