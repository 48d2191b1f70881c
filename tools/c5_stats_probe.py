import sys, time, torch
sys.path.insert(0, '.')
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200 import distributed as D
from paper_2512_04317_b200.workloads import ellipse_kspace_device
n = 16384
x = ellipse_kspace_device(n, 7, noise=0.01, rows=(0, n))
cfg = mx.PrescaleConfig()
comm = D.Comm()
res = D.compute_prescale_global(x, cfg, comm)
print("global k", res.k)
r, k = mx.prescale_stats_device(x[None], 1, n * n, cfg)
torch.cuda.synchronize()
print("device k", int(k[0]), mx.decode_results(r)[0] if hasattr(mx, 'decode_results') else '')
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
print("global ms", t(lambda: D.compute_prescale_global(x, cfg, comm)))
print("device ms", t(lambda: mx.prescale_stats_device(x[None], 1, n * n, cfg)))
