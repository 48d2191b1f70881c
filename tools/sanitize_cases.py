"""Small invocations of every hot kernel for compute-sanitizer
(racecheck / synccheck / memcheck): line passes (C2/C3/C4 shapes, columns,
transposed stores, n = 16384 rows), the fused image kernel (with and without
in-kernel statistics), the statistics kernels (lean per-segment, grid-wide
sample / count / select, the global count_range pass and the exact fallback),
the transpose kernels and the codec.  usage: python tools/sanitize_cases.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native, distributed as D  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

cfg = mx.PrescaleConfig()
for n, b, fmt, bsz in ((256, 4, "e4m3", 32), (512, 2, "e3m2", 16), (128, 6, "e4m3", 32), (64, 3, "e2m1", 64)):
    x = torch.from_numpy(ellipse_kspace_batch(b, n, seed=n, noise=0.05)).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), bsz))
    for rt in (False, True):
        mx.pipeline_device(x, p, cfg, rt)
        if n == 128:
            mx.pipeline_device(x, p, cfg, rt, fused=True)
    mx.fftcore.fft_cols_device(x, p, False)
    mx.fft2_device(x, p, "roundtrip", workspace=False)
    torch.cuda.synchronize()
    print("ok", n, fmt, bsz, flush=True)
# n = 16384 rows (one line per CTA) and the tiled transpose
p = mx.make_plan(16384, mx.ModeSpec.mx(mx.E4M3, 32))
r = (torch.randn(2, 16384, dtype=torch.complex64, device="cuda") * 2.0**-6).contiguous()
mx.fft_rows_device(r, p, False)
t = torch.randn(2, 128, 128, dtype=torch.complex64, device="cuda")
u = torch.empty_like(t)
_native.check(_native.lib().mxfft_transpose_c64(t.data_ptr(), u.data_ptr(), 2, 128, _native.stream_handle()))
# statistics: grid-wide path (few large segments), global building blocks, exact fallback
z = torch.from_numpy(ellipse_kspace_batch(1, 1024, seed=3, noise=0.01)).cuda()
mx.prescale_stats_device(z, 1, 1024 * 1024, cfg)
res = D.compute_prescale_global(z.reshape(-1), cfg, nsamples=1 << 12)
w = torch.from_numpy(ellipse_kspace_batch(3, 128, seed=9, noise=0.05)).cuda()
w[1] *= 1e-30  # extreme range: exact fallback kernel
mx.prescale_stats_device(w, 3, 128 * 128, cfg)
torch.cuda.synchronize()
print("ok stats", res.k, flush=True)
