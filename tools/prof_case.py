"""Profiling driver: runs individual passes of the C2 workload so ncu can
capture one kernel at a time.

usage: python tools/prof_case.py [rows|cols|stats|fft2|rt|fwd] [reps]
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
x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda() * (2.0 ** -14)
plan = mx.make_plan(n, mx.ModeSpec.mx(fmt, block))
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
    elif what == "fwd":
        mx.pipeline_device(x, plan, cfg, roundtrip=False, out=y)
    else:
        mx.pipeline_device(x, plan, cfg, roundtrip=True, out=y)
torch.cuda.synchronize()
print("done", what, reps)
