"""pipeline_host on the C4 headline (4096 x 128^2 round trip, graph replay): slice-weight
schemes (taper cap x slice count) against the copies-only PCIe ceiling of the box."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import mri  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

B, n = 4096, 128
x = ellipse_kspace_batch(B, n, seed=n, noise=0.05)
hx = torch.from_numpy(x).pin_memory()
hy = torch.empty(hx.shape, dtype=hx.dtype).pin_memory()
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()


def t(fn, reps=6):
    fn(); fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def make(cap):
    def host_slices(nstack, chunks):
        chunks = max(1, min(chunks, nstack))
        w = [min(cap, 2 ** i, 2 ** (chunks - 1 - i)) for i in range(chunks)]
        tot = float(sum(w))
        sizes = [max(1, int(nstack * wi / tot)) for wi in w]
        d = nstack - sum(sizes)
        order = sorted(range(chunks), key=lambda j: -w[j])
        j = 0
        while d != 0:
            k = order[j % chunks]
            if d > 0:
                sizes[k] += 1; d -= 1
            elif sizes[k] > 1:
                sizes[k] -= 1; d += 1
            j += 1
        return sizes
    return host_slices


orig = mri.host_slices
for cap in (4, 8, 16, 32):
    for chunks in (8, 10, 12, 14, 16, 20):
        mri.host_slices = make(cap)
        mri._HOST_GRAPHS.clear()
        ms = t(lambda: mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=chunks))
        print(f"cap {cap:2d} chunks {chunks:2d}: {ms:.3f} ms  {B * n * n / ms / 1e6:.2f} Gpoints/s  sizes {mri.host_slices(B, chunks)}", flush=True)
mri.host_slices = orig
