"""Which stacks does the folded pipeline leave unsettled on the bench inputs, and why?"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_04317_b200 as mx  # noqa: E402
from paper_2512_04317_b200.prescale import decode_results  # noqa: E402
from paper_2512_04317_b200.workloads import ellipse_kspace_batch  # noqa: E402

for name, batch, n, noise, fmt, b in (("c4", 4096, 128, 0.05, "e4m3", 32), ("c3", 64, 512, 0.01, "e3m2", 32),
                                      ("c2", 256, 256, 0.01, "e4m3", 32)):
    xh = ellipse_kspace_batch(batch, n, seed=n, noise=noise)
    x = torch.from_numpy(xh).cuda()
    p = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(fmt), b))
    cfg = mx.PrescaleConfig()
    y, k, res = mx.pipeline_device(x, p, cfg, True, fold=True, fused=False)
    rows = decode_results(res)
    bad = np.nonzero(rows["flags"] & 4)[0]
    _, k0, r0 = mx.pipeline_device(x, p, cfg, True, fold=False, fused=False)
    full = decode_results(r0)
    print(name, "unsettled:", bad.tolist())
    for i in bad[:8]:
        m = np.abs(xh[i].astype(np.complex128))
        mu = np.maximum(np.abs(xh[i].real), np.abs(xh[i].imag))
        mu = mu[mu > 0].min()
        L1 = np.log2(1.0 / m.max())
        print(f"  stack {i}: a_max {m.max():.6g} L1 {L1:.7f} k1 {full['k1'][i]} k2 {full['k2'][i]} k {full['k'][i]} "
              f"p_tau {full['p_tau'][i]:.4g} min nonzero max(|re|,|im|) {mu:.4g}  bound 2 tau_min 2^-k1 "
              f"{2 * cfg.tau_min * 2.0 ** -int(full['k1'][i]):.4g} zeros {(m == 0).sum()}")
