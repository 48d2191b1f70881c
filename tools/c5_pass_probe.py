"""One n = 16384 forward fft2 (split passes) after a warm-up, for an ncu launch list."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_device  # noqa: E402

n = 16384
x = ellipse_kspace_device(n, 7) * (2.0 ** -20)
p = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
for _ in range(3):
    y = mx.fft2_device(x[None], p, "forward")
torch.cuda.synchronize()
print("done")
