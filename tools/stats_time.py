"""Statistics kernel time at the C4 / C2 / C3 shapes (CUDA events, 20 reps); the
library under test comes from MXFFT_B200_LIB (A/B of builds)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200.workloads import ellipse_kspace_batch
cfg = mx.PrescaleConfig()
shapes = ((128, 4096, 0.05), (256, 256, 0.01), (512, 64, 0.01))
if len(sys.argv) > 1:
    shapes = shapes[:int(sys.argv[1])]
for n, batch, noise in shapes:
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=1000 + n, noise=noise)).cuda()
    for _ in range(3):
        k, res = mx.prescale_stats_device(x, batch, n * n, cfg)[:2]
    torch.cuda.synchronize()
    ts = []
    for rnd in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20):
            mx.prescale_stats_device(x, batch, n * n, cfg)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 20 * 1e3)
    print(f"stats n={n} batch={batch}: {sorted(ts)[2]:.1f} us (min {min(ts):.1f})")
