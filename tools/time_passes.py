"""Quick per-kernel timing of the C2 workload (CUDA events, warm, averaged).
usage: python tools/time_passes.py [n] [batch] [fmt] [B]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 256
fmt = mx.get_mx_format(sys.argv[3] if len(sys.argv) > 3 else "e4m3")
B = int(sys.argv[4]) if len(sys.argv) > 4 else 32
x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda()
plan = mx.make_plan(n, mx.ModeSpec.mx(fmt, B))
y = torch.empty_like(x)
cfg = mx.PrescaleConfig()
k = torch.empty(batch, dtype=torch.int32, device="cuda")
r = torch.empty((batch, 40), dtype=torch.uint8, device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


pts = batch * n * n
res = {
    "rows_us": t(lambda: mx.fft_rows_device(x, plan, False, out=y)),
    "cols_us": t(lambda: mx.fftcore.fft_cols_device(x, plan, False, out=y)),
    "stats_us": t(lambda: mx.prescale_stats_device(x, batch, n * n, cfg, k_out=k, res_out=r)),
    "fwd_us": t(lambda: mx.pipeline_device(x, plan, cfg, False, out=y, k=k, res=r)),
    "rt_us": t(lambda: mx.pipeline_device(x, plan, cfg, True, out=y, k=k, res=r)),
}
res["rt_gpts"] = pts / res["rt_us"] / 1e3
res["fwd_gpts"] = pts / res["fwd_us"] / 1e3
res["pass_GBs"] = 16 * pts / min(res["rows_us"], res["cols_us"]) / 1e3
print(f"n={n} batch={batch} {fmt.name} B={B}: " + " ".join(f"{k}={v:.1f}" for k, v in res.items()))
