"""PCIe probe for the host-buffer pipeline: pinned H2D / D2H bandwidth alone
and concurrently, and pipeline_host (C2 round trip) over several slice counts.
usage: python tools/pcie_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

nb = 256 * 256 * 256 * 8
h = torch.empty(nb, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


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


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = t(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {nb / ms / 1e6:.1f} GB/s")
ms = t(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {nb / ms / 1e6:.1f} GB/s")
ms = t(both)
print(f"H2D+D2H concurrent {nb / ms / 1e6:.1f} GB/s each")
for chunk in (1 << 20, 4 << 20, 16 << 20):
    def many():
        for o in range(0, nb, chunk):
            d[o:o + chunk].copy_(h[o:o + chunk], non_blocking=True)
    ms = t(many)
    print(f"H2D in {chunk >> 20} MiB pieces {nb / ms / 1e6:.1f} GB/s")

x = ellipse_kspace_batch(256, 256, seed=0)
hx = torch.from_numpy(x).pin_memory()
hy = torch.empty_like(hx).pin_memory()
plan = mx.make_plan(256, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
for ch in (4, 8, 16, 32, 64):
    ms = t(lambda: mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=ch))
    print(f"pipeline_host chunks={ch}: {ms:.3f} ms  {256 * 65536 / ms / 1e6:.2f} Gpoints/s")

# enqueue cost of one slice's compute (host-side Python + C-ABI launches)
import time  # noqa: E402

xs = torch.from_numpy(x[:32]).cuda()
ys = torch.empty_like(xs)
kk = torch.empty(32, dtype=torch.int32, device="cuda")
for _ in range(3):
    mx.pipeline_device(xs, plan, cfg, True, out=ys, k=kk)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    mx.pipeline_device(xs, plan, cfg, True, out=ys, k=kk)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"pipeline_device(32 imgs) enqueue {1e3 * (t1 - t0) / 50:.3f} ms/call, total {1e3 * (t2 - t0) / 50:.3f} ms/call")
t0 = time.perf_counter()
for _ in range(20):
    mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=8)
print(f"pipeline_host chunks=8 wall {1e3 * (time.perf_counter() - t0) / 20:.3f} ms/call")
