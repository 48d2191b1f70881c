"""Profiling driver: runs individual passes of the C2 workload so ncu can
capture one kernel at a time.

usage: python tools/prof_case.py [rows|cols|stats|fft2|rtk|rt|fwd] [reps]
env:   PROF_N (256), PROF_BATCH (256), PROF_FMT (e4m3), PROF_B (32)
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "rows"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(os.environ.get("PROF_N", "256"))
batch = int(os.environ.get("PROF_BATCH", "256"))
fmt = mx.get_mx_format(os.environ.get("PROF_FMT", "e4m3"))
block = int(os.environ.get("PROF_B", "32"))
if n >= 8192:  # the host generator would take minutes at this size
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    x = torch.stack([ellipse_kspace_device(n, 7 + i) for i in range(batch)]) * (2.0 ** -14)
else:
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda() * (2.0 ** -14)
plan = mx.make_plan(n, mx.ModeSpec.mx(fmt, block))
if os.environ.get("MXFFT_FUSED_IMAGE") == "0":  # n = 128: profile the line passes instead of the fused kernel
    mx._native.lib().mxfft_fused_image(0)
y = torch.empty_like(x)
cfg = mx.PrescaleConfig()
for _ in range(reps):
    if what == "rows":
        mx.fft_rows_device(x, plan, False, out=y)
    elif what == "cols":
        mx.fftcore.fft_cols_device(x, plan, False, out=y)
    elif what == "stats":
        mx.prescale_stats_device(x, batch, n * n, cfg)
    elif what == "fft2":
        mx.fft2_device(x, plan, "forward", out=y)
    elif what == "rtk":  # the 4-pass round trip with per-image k (the C4 headline's transform)
        kk = torch.full((batch,), -12, dtype=torch.int32, device="cuda")
        mx.fft2_device(x * (2.0 ** 14), plan, "roundtrip", k=kk, out=y)
    elif what == "fwd":
        mx.pipeline_device(x, plan, cfg, roundtrip=False, out=y)
    else:
        mx.pipeline_device(x, plan, cfg, roundtrip=True, out=y)
torch.cuda.synchronize()
print("done", what, reps)
