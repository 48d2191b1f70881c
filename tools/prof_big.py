"""One n = 16384 row pass (C5 geometry) on random data, for ncu.  usage: python tools/prof_big.py [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402

n = 16384
x = torch.randn(n, n, dtype=torch.complex64, device="cuda")
y = torch.empty_like(x)
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    mx.fft_rows_device(x, plan, False, out=y)
torch.cuda.synchronize()
