"""How often does the sampled statistics path settle a segment?  Runs
prescale_stats_device on the BASELINE batch shapes and reports how many
segments went to the exact fallback kernel (the work list the fast path
leaves in its workspace: SegState[nseg] | int list[nseg] + count)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200 import _native  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

for n, b in ((256, 256), (512, 64), (128, 4096), (256, 8)):
    x = torch.from_numpy(ellipse_kspace_batch(b, n, seed=0)).cuda()
    need = int(_native.load().mxfft_prescale_workspace_bytes(b, n * n))
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    mx.prescale_stats_device(x, b, n * n, mx.PrescaleConfig(), workspace=ws)
    torch.cuda.synchronize()
    off = (40 * b + 255) // 256 * 256
    lst = ws[off: off + 4 * (b + 1)].view(torch.int32).cpu()
    print(f"n={n} batch={b}: {int(lst[b])} of {b} segments settled by the exact fallback")
