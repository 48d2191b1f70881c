"""Graph-replayed round-trip pipelines (fold on / off) at the C4 / C2 / C3 shapes; ms per step."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cases = (("c4", 4096, 128, 0.05, "e4m3", 32), ("c2", 256, 256, 0.01, "e4m3", 32), ("c3", 64, 512, 0.01, "e3m2", 32),
         ("c1", 1, 256, 0.01, "e4m3", 32))
reps = int(os.environ.get("REPS", "3"))
for name, batch, n, noise, fmt, b in cases:
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=n, noise=noise)).cuda()
    y = torch.empty_like(x)
    k = torch.empty(batch, dtype=torch.int32, device="cuda")
    res = torch.empty((batch, 40), dtype=torch.uint8, device="cuda")
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), b))
    cfg = mx.PrescaleConfig()
    mx._native.lib().mxfft_fused_image(0)
    out = []
    for fold in (False, True) * reps:
        f = lambda: mx.pipeline_device(x, p, cfg, True, out=y, k=k, res=res, fused=False, fold=fold)
        f(); f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            f()
        ts = []
        for i in range(25):
            flush_buf.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1))
        out.append((fold, sum(ts) / len(ts)))
    print(name, " ".join(f"{'fold' if f else 'std'} {t * 1e3:.1f}" for f, t in out), flush=True)
