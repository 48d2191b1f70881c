"""Time mxfft_fft2 (forward / round trip) with and without the transposed-store
workspace, optionally at a stage cap (profiling only).
usage: python tools/time_fft2.py [n] [batch] [stage_limit]"""
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
lim = int(sys.argv[3]) if len(sys.argv) > 3 else -1
x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda() * (2.0 ** -14)
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
y = torch.empty_like(x)
ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, batch)),
                 dtype=torch.uint8, device="cuda")
_native.lib().mxfft_profile_stage_limit(lim)


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


for mode in ("forward", "roundtrip"):
    a = t(lambda: mx.fft2_device(x, plan, mode, out=y, workspace=ws))
    b = t(lambda: mx.fft2_device(x, plan, mode, out=y, workspace=False))
    npass = 2 if mode == "forward" else 4
    print(f"n={n} batch={batch} lim={lim} {mode:9s}: transposed-store {a:8.1f} us "
          f"({a / npass:6.1f}/pass)  in-place cols {b:8.1f} us ({b / npass:6.1f}/pass)")
_native.lib().mxfft_profile_stage_limit(-1)
