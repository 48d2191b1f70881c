"""Multi-rank orchestration (paper_2512_04317_b200/distributed.py) on CPU:
the global prescale over a segment split across ranks, and the row-slab 2-D
transform with all-to-all transposes, against the single-process oracle.
Ranks talk over gloo (world size 2 and 4, 127.0.0.1); the per-rank compute
is the oracle stand-in tests/cpu_ops.py (the CUDA primitives are covered by
the gpu tests)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O
from cpu_ops import OracleOps, SlabPlan
from paper_2512_04317_b200 import distributed as D
from paper_2512_04317_b200.prescale import PrescaleConfig
from paper_2512_04317_b200.workloads import ellipse_kspace


def test_shard_range_partitions():
    for n in (0, 1, 7, 256, 4097):
        for w in (1, 2, 3, 8):
            parts = [D.shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard_range(4, 2, 2)


def _oracle_prescale(x):
    r = O.compute_prescale(x)
    return r.a_max, r.p_tau, r.k1, r.k2, r.k


@pytest.mark.parametrize("n,seed,noise", [(128, 0, 0.01), (256, 1, 0.05), (64, 2, 0.0)])
def test_global_prescale_single_process_matches_oracle(n, seed, noise):
    x = ellipse_kspace(n, seed, noise=noise) * np.float32(2.0**-3)
    got = D.compute_prescale_global(torch.from_numpy(x.reshape(-1)), PrescaleConfig(), ops=OracleOps(),
                                    nsamples=1 << 12)
    a_max, p_tau, k1, k2, k = _oracle_prescale(x)
    assert (got.k, got.k1, got.k2) == (k, k1, k2)
    assert got.a_max == a_max and got.p_tau == p_tau


def test_global_prescale_tiny_sample_widens_bracket():
    """A 16-key sample gives a bracket that misses the quantile; the widening
    retries must still land on the exact statistics."""
    x = ellipse_kspace(64, 5, noise=0.02)
    got = D.compute_prescale_global(torch.from_numpy(x.reshape(-1)), PrescaleConfig(), ops=OracleOps(),
                                    nsamples=16)
    a_max, p_tau, k1, k2, k = _oracle_prescale(x)
    assert (got.k, got.a_max, got.p_tau) == (k, a_max, p_tau)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, seed, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.Comm()
        ops = OracleOps()
        plan = SlabPlan(n)
        x = ellipse_kspace(n, seed, noise=0.01).astype(np.complex64)
        r0, r1 = D.shard_range(n, rank, world)
        slab = torch.from_numpy(np.ascontiguousarray(x[r0:r1]))
        res = D.compute_prescale_global(slab, PrescaleConfig(), comm, ops, nsamples=1 << 10)
        fwd = D.fft2_slab(slab, plan, "forward", comm, ops).numpy()
        fwd_t = D.fft2_slab(slab, plan, "forward", comm, ops, restore=False).numpy()
        inv = D.fft2_slab(slab, plan, "inverse", comm, ops).numpy()
        rt, res2 = D.pipeline_slab(slab, plan, PrescaleConfig(), True, comm, ops, fold=False)
        # the folded prescale: first pass with evidence, two all-reduces, every rank the same k
        rt_f, res_f = D.pipeline_slab(slab, plan, PrescaleConfig(), True, comm, ops, fold=True)
        # a configuration in which k2 wins: the fold declines on every rank and the statistics path runs
        cfg2 = PrescaleConfig(tau_min=0.5)
        rt_d, res_d = D.pipeline_slab(slab, plan, cfg2, True, comm, ops, fold=True)
        res_s = D.compute_prescale_global(slab, cfg2, comm, ops, nsamples=1 << 10)
        q.put((rank, r0, r1, res, fwd, fwd_t, inv, rt.numpy(), res2, rt_f.numpy(), res_f, res_d, res_s))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_row_slabs_gloo_match_single_image_oracle(world):
    n, seed = 64, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o[0])
    x = ellipse_kspace(n, seed, noise=0.01).astype(np.complex64)
    oplan = O.make_plan(n, O.E4M3, 32)
    a_max, p_tau, k1, k2, k = _oracle_prescale(x)
    f = O.fft2(x, oplan, False)
    fi = O.fft2(x, oplan, True)
    out_o, _, k_o = O.pipeline(x, oplan, True)
    for rank, r0, r1, res, fwd, fwd_t, inv, rt, res2, rt_f, res_f, res_d, res_s in outs:
        assert res_f.k == k_o and np.isnan(res_f.p_tau)  # settled by the fold (k-only result)
        np.testing.assert_array_equal(rt_f.astype(np.complex128), out_o[0][r0:r1])
        assert res_d.k == res_s.k and res_d.p_tau == res_s.p_tau and res_s.k2 > res_s.k1  # declined -> statistics
        assert (res.k, res.a_max, res.p_tau) == (k, a_max, p_tau)
        assert res2.k == k_o
        np.testing.assert_array_equal(fwd, f[r0:r1])
        np.testing.assert_array_equal(fwd_t, f.T[r0:r1])
        np.testing.assert_array_equal(inv, fi[r0:r1])
        np.testing.assert_array_equal(rt.astype(np.complex128), out_o[0][r0:r1])
