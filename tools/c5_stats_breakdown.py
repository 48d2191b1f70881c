"""Time the steps of distributed.compute_prescale_global on the C5 image (1 GPU)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200 import distributed as D
from paper_2512_04317_b200.workloads import ellipse_kspace_device
n = 16384
x = ellipse_kspace_device(n, 7, noise=0.01, rows=(0, n)).reshape(-1)
cfg = mx.PrescaleConfig()
ops = D.CudaOps()
q = cfg.tau / 100.0
def T(label, fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): r = fn()
    torch.cuda.synchronize()
    print(f"{label:28s} {(time.perf_counter() - t0) / reps * 1e3:8.3f} ms", flush=True)
    return r
keys = T("sample_keys 2^18", lambda: ops.sample_keys(x, 1 << 18))
sk = T("sort keys", lambda: torch.sort(keys).values)
hk = T("keys .cpu()", lambda: sk.cpu().numpy())
lo, hi, top, nsamp = D._bracket(hk, q, 1.0)
f = (min(nsamp, int(np.searchsorted(hk[:nsamp], hi, side="right"))) - int(np.searchsorted(hk[:nsamp], lo, side="left"))) / nsamp
npts = x.numel()
cap = min(npts, int(npts * f * 2) + 65536); tcap = min(npts, int(4 * npts / nsamp) + 4096)
print("bracket fraction", f, "cand cap", cap)
out = T("count_range", lambda: ops.count_range(x, float(lo), float(hi), float(top), cap, tcap))
(nnz, below, ncand, ntop, flags), cand, topb = out
print("ncand", int(ncand), "ntop", int(ntop))
c = T("cabs(cand)", lambda: ops.cabs(cand))
T("sort mags", lambda: torch.sort(c).values)
T("full global", lambda: D.compute_prescale_global(x, cfg))
