"""n = 8192 / 16384 passes: plain row pass vs transposed-store fft2 pass vs
in-place column pass.  usage: python tools/time_big.py [n]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
x = torch.cat([ellipse_kspace_device(n, 7 + i) for i in range(batch)]) * (2.0 ** -20)
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
y = torch.empty_like(x)
ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, batch)), dtype=torch.uint8,
                 device="cuda")


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


gb = batch * n * n * 16 / 1e9
for name, fn, npass in (("rows", lambda: mx.fft_rows_device(x, plan, False, out=y), 1),
                        ("cols in place", lambda: mx.fftcore.fft_cols_device(x.view(batch, n, n), plan, False,
                                                                            out=y.view(batch, n, n)), 1),
                        ("fft2 (current)", lambda: mx.fft2_device(x.view(batch, n, n), plan, "forward",
                                                                 out=y.view(batch, n, n), workspace=ws), 2),
                        ("mxfft transpose", lambda: _native.check(_native.lib().mxfft_transpose_c64(
                            x.data_ptr(), y.data_ptr(), batch, n, _native.stream_handle())), 1)):
    ms = t(fn) / npass
    print(f"n={n} batch={batch} {name:16s} {ms:8.3f} ms/pass  {gb / ms * 1e3:7.0f} GB/s")
