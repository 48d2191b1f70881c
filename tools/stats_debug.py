"""How often does the sampled statistics path settle a segment?"""
import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200 import _native
from paper_2512_04317_b200.workloads import ellipse_kspace_batch
for n, b in ((256, 256), (512, 64), (128, 4096)):
    x = torch.from_numpy(ellipse_kspace_batch(b, n, seed=0)).cuda()
    cfg = mx.PrescaleConfig()
    need = int(_native.load().mxfft_prescale_workspace_bytes(b, n * n))
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    mx.prescale_stats_device(x, b, n * n, cfg, workspace=ws)
    torch.cuda.synchronize()
    st = ws[: 40 * b].view(torch.int32).view(b, 10).cpu().numpy()
    stf = ws[: 40 * b].view(torch.float32).view(b, 10).cpu().numpy()
    fb_off = ((40 * b + 255) // 256) * 256
    fb = ws[fb_off: fb_off + 4 * b].view(torch.int32).cpu().numpy()
    print(f"n={n} b={b}: fallback {fb.sum()}/{b}; ncand mean {st[:, 7].mean():.0f} max {st[:, 7].max()}; ntop max {st[:, 8].max()}; flags {np.unique(st[:, 9])}; below mean {st[:,6].mean():.0f}; nnz {st[:,4].mean():.0f}")
    print("  lo/hi/top img0:", stf[0, :3], " cand:", st[0, 7], "below:", st[0, 6])
