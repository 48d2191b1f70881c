"""pipeline_host (C4 e2e) with different slice counts."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

x = ellipse_kspace_batch(4096, 128, seed=0, noise=0.05)
p = mx.make_plan(128, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
h = torch.from_numpy(x).pin_memory()
o = torch.empty_like(h).pin_memory()
for chunks in (4, 8, 12, 16, 24, 32):
    f = lambda: mx.pipeline_host(h, p, cfg, True, out_host=o, chunks=chunks)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"chunks={chunks:3d} {ms:7.3f} ms/step  {4096 * 128 * 128 / ms / 1e6:6.2f} Gpt/s", flush=True)
