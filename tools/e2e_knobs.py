"""e2e (pipeline_host, pinned buffers, 12 slices) under the scheduling knobs."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_04317_b200 as mx
from paper_2512_04317_b200 import _native
from paper_2512_04317_b200.workloads import ellipse_kspace_batch
L = _native.lib()
n, batch = 128, 4096
x = ellipse_kspace_batch(batch, n, seed=1128, noise=0.05)
h_in = torch.from_numpy(x).pin_memory()
h_out = torch.empty(h_in.shape, dtype=h_in.dtype).pin_memory()
plan = mx.make_plan(n, mx.ModeSpec.mx(mx.E4M3, 32))
cfg = mx.PrescaleConfig()
for fused, pdl, tma in ((1, 1, 1), (-1, 0, 1), (-1, 1, 1), (0, 1, 0), (-1, 1, 1)):
    L.mxfft_fused_image(fused); L.mxfft_pdl(pdl); L.mxfft_tma_store(tma)
    mx.mri._HOST_GRAPHS.clear() if hasattr(mx.mri, "_HOST_GRAPHS") else None
    for _ in range(2):
        mx.pipeline_host(h_in, plan, cfg, True, out_host=h_out, chunks=12)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        mx.pipeline_host(h_in, plan, cfg, True, out_host=h_out, chunks=12)
    e1.record(); torch.cuda.synchronize()
    print(f"fused={fused} pdl={pdl} tma={tma}: {e0.elapsed_time(e1)/5:.2f} ms/step")
