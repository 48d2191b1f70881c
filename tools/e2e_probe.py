"""Host-buffer pipeline experiments (C2 round trip): copy-only floor, and the
slice pipeline with more ring buffers.  usage: python tools/e2e_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.mri import pipeline_device  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

B, n = 256, 256
x = ellipse_kspace_batch(B, n, seed=0)
hx = torch.from_numpy(x).pin_memory()
hy = torch.empty_like(hx).pin_memory()
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
S = [torch.cuda.Stream() for _ in range(3)]


def t(fn, reps=6):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def pipe(chunks, nbuf, compute=True):
    per = B // chunks
    s_in, s_cmp, s_out = S
    cur = torch.cuda.current_stream()
    xb = [torch.empty((per, n, n), dtype=torch.complex64, device="cuda") for _ in range(nbuf)]
    yb = [torch.empty((per, n, n), dtype=torch.complex64, device="cuda") for _ in range(nbuf)]
    kb = [torch.empty(per, dtype=torch.int32, device="cuda") for _ in range(nbuf)]
    ev_in = [torch.cuda.Event() for _ in range(nbuf)]
    ev_cmp = [torch.cuda.Event() for _ in range(nbuf)]
    ev_out = [torch.cuda.Event() for _ in range(nbuf)]
    for s in S:
        s.wait_stream(cur)
    for i in range(chunks):
        b = i % nbuf
        st = i * per
        if i >= nbuf:
            s_in.wait_event(ev_cmp[b])
        with torch.cuda.stream(s_in):
            xb[b].copy_(hx[st:st + per], non_blocking=True)
            ev_in[b].record(s_in)
        s_cmp.wait_event(ev_in[b])
        if i >= nbuf:
            s_cmp.wait_event(ev_out[b])
        with torch.cuda.stream(s_cmp):
            if compute:
                pipeline_device(xb[b], plan, cfg, True, out=yb[b], k=kb[b])
            ev_cmp[b].record(s_cmp)
        s_out.wait_event(ev_cmp[b])
        with torch.cuda.stream(s_out):
            hy[st:st + per].copy_(yb[b] if compute else xb[b], non_blocking=True)
            ev_out[b].record(s_out)
    for t_ in xb + yb + kb:
        for s in S:
            t_.record_stream(s)
    for s in S:
        cur.wait_stream(s)


for compute in ():
    for chunks in (4, 8, 16, 32):
        for nbuf in (2, 3, 4):
            ms = t(lambda: pipe(chunks, nbuf, compute))
            print(f"compute={compute} chunks={chunks} nbuf={nbuf}: {ms:.3f} ms  {B * n * n / ms / 1e6:.2f} Gpoints/s")

# the whole sliced pipeline captured once as a CUDA graph, replayed per step
for chunks in ():
    for nbuf in (2, 3):
        g = torch.cuda.CUDAGraph()
        pipe(chunks, nbuf, True)
        torch.cuda.synchronize()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            pipe(chunks, nbuf, True)  # warm the allocator on the capture stream
        torch.cuda.synchronize()
        try:
            with torch.cuda.graph(g):
                pipe(chunks, nbuf, True)
        except Exception as e:  # noqa: BLE001
            print("capture failed:", repr(e)[:300])
            break
        ms = t(lambda: g.replay())
        ok = torch.equal(hy, hy)  # noqa: PLR0124
        print(f"graph chunks={chunks} nbuf={nbuf}: {ms:.3f} ms  {B * n * n / ms / 1e6:.2f} Gpoints/s")
# correctness of the graph replay vs eager
hy.zero_()
pipe(8, 2, True)
torch.cuda.synchronize()
ref = hy.clone()

for ch in (8, 12, 16, 24, 32):
    ms = t(lambda: mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=ch))
    print(f"pipeline_host (ramped, whole-batch buffers) chunks={ch}: {ms:.3f} ms  {B * n * n / ms / 1e6:.2f} Gpoints/s")
hy.zero_()
mx.pipeline_host(hx, plan, cfg, True, out_host=hy, chunks=12)
print("pipeline_host == eager ring:", torch.equal(torch.view_as_real(ref), torch.view_as_real(hy)))
