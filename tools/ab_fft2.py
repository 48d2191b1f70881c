"""A/B timing of several builds of libmxfft_b200.so in one process: each build
gets its own plan; mxfft_fft2 (forward, transposed-store workspace) is timed
round-robin over several rounds so clock drift and box noise hit every build
alike.  usage: python tools/ab_fft2.py n batch lib1.so [lib2.so ...]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_04317_b200 import _native, fftcore  # noqa: E402
from paper_2512_04317_b200.minifloat import E4M3  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

n, batch = int(sys.argv[1]), int(sys.argv[2])
libs = sys.argv[3:]
if n >= 8192:  # the host generator would take minutes at this size
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    x = torch.stack([ellipse_kspace_device(n, 7 + i) for i in range(batch)]) * (2.0 ** -14)
else:
    x = torch.from_numpy(ellipse_kspace_batch(batch, n, seed=0)).cuda() * (2.0 ** -14)
y = torch.empty_like(x)
tw = np.ascontiguousarray(np.stack(fftcore._twiddle_table(n)))
c = E4M3.as_c()
runs = []
for path in libs:
    L = ctypes.CDLL(path)
    for name, (argt, rest) in _native.SIGNATURES.items():
        if hasattr(L, name):
            getattr(L, name).argtypes = argt
            getattr(L, name).restype = rest
    if hasattr(L, "mxfft_fused_image"):
        L.mxfft_fused_image(int(os.environ.get("AB_FUSED", "0")))  # A/B the line passes unless asked
    h = ctypes.c_void_p()
    assert L.mxfft_plan_create(ctypes.byref(h), n, ctypes.byref(c), 32, tw.ctypes.data, 0) == 0
    wsb = int(L.mxfft_fft2_workspace_bytes(h, batch))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    runs.append((os.path.basename(os.path.dirname(path)), L, h, ws, wsb))

stream = torch.cuda.current_stream().cuda_stream
mode = int(os.environ.get("AB_MODE", "0"))  # 0 forward, 2 round trip (timed per pass either way)
npass = 4 if mode == 2 else 2
kk = torch.full((batch,), -3, dtype=torch.int32, device="cuda") if os.environ.get("AB_K") else None


def t(L, h, ws, wsb, reps=30):
    f = lambda: L.mxfft_fft2(h, x.data_ptr(), y.data_ptr(), batch, mode, kk.data_ptr() if kk is not None else None, 1, ws.data_ptr(), wsb, stream)
    for _ in range(3):
        assert f() == 0
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3 / npass  # per pass


res = {r[0]: [] for r in runs}
outs = {}
for rnd in range(5):
    for name, L, h, ws, wsb in runs:
        res[name].append(t(L, h, ws, wsb))
        if rnd == 0:
            outs[name] = y.clone()
base = runs[0][0]
for name in res:
    v = sorted(res[name])
    same = torch.equal(torch.view_as_real(outs[name]), torch.view_as_real(outs[base]))
    print(f"n={n} batch={batch} {name:12s} us/pass median {v[len(v) // 2]:7.1f}  min {v[0]:7.1f}  "
          f"max {v[-1]:7.1f}  same-as-{base}: {same}")
