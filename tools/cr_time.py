"""Time the global statistics' count pass on the C5 image (CUDA events, 20 reps)."""
import sys
import torch
sys.path.insert(0, '.')
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200 import distributed as D
from paper_2512_04317_b200.workloads import ellipse_kspace_device
n = 16384
x = ellipse_kspace_device(n, 7, noise=0.01, rows=(0, n)).reshape(-1)
ops = D.CudaOps()
cfg = mx.PrescaleConfig()
keys = torch.sort(ops.sample_keys(x, 1 << 18)).values
nf = int(torch.isfinite(keys).sum())
lo, hi, top, ns = D._bracket_dev(keys, nf, cfg.tau / 100.0, 1.0)
f = lambda: ops.count_range(x, float(lo), float(hi), float(top), 940032, 20000)
r = f(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20): f()
e1.record(); torch.cuda.synchronize()
print(f"count_range {e0.elapsed_time(e1) / 20:.3f} ms  ncand {int(r[0][2])}")
g = lambda: D.compute_prescale_global(x.reshape(n, n), cfg)
g(); torch.cuda.synchronize()
e0.record()
for _ in range(10): g()
e1.record(); torch.cuda.synchronize()
print(f"global {e0.elapsed_time(e1) / 10:.3f} ms")
