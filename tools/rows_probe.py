"""Row-pass cost per point for large n on 2^28 points (C5 restructuring probe):
python tools/rows_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native  # noqa: E402

L = _native.lib()
g = torch.Generator(device="cuda")
g.manual_seed(0)
N = 1 << 28
x = torch.complex(torch.randn(N, generator=g, device="cuda"), torch.randn(N, generator=g, device="cuda")) * 2.0**-4
y = torch.empty_like(x)


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


for n in (2048, 4096, 8192, 16384):
    plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
    xr, yr = x.view(-1, n), y.view(-1, n)
    for cps in (0, 1, 2, 3, 4):
        L.mxfft_lines_ctas_per_sm(cps)
        ms = t(lambda: mx.fft_rows_device(xr, plan, False, out=yr))
        print(f"n={n:6d} stages={n.bit_length()-1:2d} ctas/sm cap={cps}: {ms:7.3f} ms per 2^28-point pass, "
              f"{ms / (n.bit_length()-1):6.3f} ms per stage")
    L.mxfft_lines_ctas_per_sm(0)
