"""Would the prescale statistics hide behind the first line pass?  Times (C2):
stats alone, the forward row pass alone at 3 and 2 CTAs/SM, and both launched
together on two streams.  usage: python tools/concurrency_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

B, n = 256, 256
x = torch.from_numpy(ellipse_kspace_batch(B, n, seed=0)).cuda()
y = torch.empty_like(x)
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
L = _native.lib()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def stats():
    with torch.cuda.stream(sa):
        mx.prescale_stats_device(x, B, n * n, cfg)


def rows():
    with torch.cuda.stream(sb):
        mx.fft_rows_device(x, plan, False, out=y)


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        sa.wait_stream(torch.cuda.current_stream())
        sb.wait_stream(torch.cuda.current_stream())
        fn()
        torch.cuda.current_stream().wait_stream(sa)
        torch.cuda.current_stream().wait_stream(sb)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print(f"stats alone {t(stats):.1f} us")
for c in (0, 2, 1):
    L.mxfft_lines_ctas_per_sm(c)
    print(f"ctas/SM={c or 'occ'}: rows alone {t(rows):.1f} us; stats then rows {t(lambda: (stats(), sb.wait_stream(sa), rows())):.1f} us; "
          f"stats || rows {t(lambda: (stats(), rows())):.1f} us; rows || stats {t(lambda: (rows(), stats())):.1f} us")
L.mxfft_lines_ctas_per_sm(0)
