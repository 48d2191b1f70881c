"""A/B timing of the prescale statistics of several libmxfft_b200.so builds in
one process (round-robin, like ab_fft2.py); results must be identical.
usage: python tools/ab_stats.py n batch lib1.so [lib2.so ...]"""
import ctypes
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_04317_b200 import _native  # noqa: E402
from paper_2512_04317_b200.prescale import PrescaleConfig  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

n, batch = int(sys.argv[1]), int(sys.argv[2])
libs = sys.argv[3:]
x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda()
c = PrescaleConfig().as_c()
stream = torch.cuda.current_stream().cuda_stream
runs = []
for path in libs:
    L = ctypes.CDLL(path)
    for name, (argt, rest) in _native.SIGNATURES.items():
        if hasattr(L, name):
            getattr(L, name).argtypes = argt
            getattr(L, name).restype = rest
    need = int(L.mxfft_prescale_workspace_bytes(batch, n * n))
    ws = torch.zeros(max(need, 1), dtype=torch.uint8, device="cuda")
    res = torch.zeros((batch, 40), dtype=torch.uint8, device="cuda")
    k = torch.zeros(batch, dtype=torch.int32, device="cuda")
    runs.append((os.path.basename(os.path.dirname(path)), L, ws, need, res, k))


def t(L, ws, need, res, k, reps=30):
    f = lambda: L.mxfft_prescale_stats(x.data_ptr(), 0, batch, n * n, ctypes.byref(c), res.data_ptr(),  # noqa: E731
                                       k.data_ptr(), ws.data_ptr(), need, stream)
    for _ in range(3):
        assert f() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


tm = {r[0]: [] for r in runs}
for rnd in range(5):
    for name, L, ws, need, res, k in runs:
        tm[name].append(t(L, ws, need, res, k))
base = runs[0][4]
for name, L, ws, need, res, k in runs:
    v = sorted(tm[name])
    print(f"n={n} batch={batch} {name:12s} us median {v[len(v) // 2]:7.1f} min {v[0]:7.1f}  "
          f"same-as-first: {torch.equal(res, base)}")
