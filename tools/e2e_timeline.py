"""Event timeline of pipeline_host-style slicing (C2 round trip): when each
slice's H2D / compute / D2H starts and ends.  usage: python tools/e2e_timeline.py [chunks]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.mri import pipeline_device  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

B, n = int(os.environ.get("TL_B", "256")), int(os.environ.get("TL_N", "256"))
chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
x = ellipse_kspace_batch(B, n, seed=0)
hx = torch.from_numpy(x).pin_memory()
hy = torch.empty_like(hx).pin_memory()
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
S = [torch.cuda.Stream() for _ in range(3)]
from paper_2512_04317_b200.mri import host_slices  # noqa: E402

sizes = host_slices(B, chunks)
starts = [sum(sizes[:i]) for i in range(len(sizes))]
X = torch.empty((B, n, n), dtype=torch.complex64, device="cuda")
Y = torch.empty_like(X)
K = torch.empty(B, dtype=torch.int32, device="cuda")


def run(tl):
    s_in, s_cmp, s_out = S
    cur = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    e_in = [ev() for _ in range(2)]
    e_cmp = [ev() for _ in range(2)]
    e_out = [ev() for _ in range(2)]
    t0 = ev()
    t0.record(cur)
    for s in S:
        s.wait_stream(cur)
    for i in range(len(sizes)):
        b = i & 1
        st, per = starts[i], sizes[i]
        xb, yb, kb = {b: X[st:st + per]}, {b: Y[st:st + per]}, {b: K[st:st + per]}
        a = ev(); a.record(s_in)
        with torch.cuda.stream(s_in):
            xb[b].copy_(hx[st:st + per], non_blocking=True)
        e_in[b] = ev(); e_in[b].record(s_in)
        s_cmp.wait_event(e_in[b])
        c = ev(); c.record(s_cmp)
        with torch.cuda.stream(s_cmp):
            pipeline_device(xb[b], plan, cfg, True, out=yb[b], k=kb[b])
        e_cmp[b] = ev(); e_cmp[b].record(s_cmp)
        s_out.wait_event(e_cmp[b])
        d = ev(); d.record(s_out)
        with torch.cuda.stream(s_out):
            hy[st:st + per].copy_(yb[b], non_blocking=True)
        e_out[b] = ev(); e_out[b].record(s_out)
        tl.append((a, e_in[b], c, e_cmp[b], d, e_out[b]))
    for s in S:
        cur.wait_stream(s)
    return t0


for rep in range(3):
    tl = []
    t0 = run(tl)
    torch.cuda.synchronize()
print("slice  h2d[start end]   cmp[start end]   d2h[start end]  (ms from step start)")
for i, evs in enumerate(tl):
    ts = [t0.elapsed_time(e) for e in evs]
    print(f"{i:3d}  " + "   ".join(f"{ts[j]:6.3f} {ts[j + 1]:6.3f}" for j in (0, 2, 4)))
