"""MX-FFT2 benchmark (BASELINE.json metric) on N GPUs of one node.

Workload (BASELINE.json configs[1], "C2"): a batch of 256 seeded synthetic
k-space images, 256 x 256 complex64 each (ellipse phantoms + 1% complex
Gaussian noise, paper_2512_04317_b200/workloads.py), MXFP8 E4M3, B = 32.
One step = the round-trip pipeline over the whole batch, entirely on the GPU:
per-image prescale statistics (amax + tau-percentile radix-select, k on
device) -> forward MX-FFT2 with x*2^k fused into the first load -> inverse
MX-FFT2 -> x 2^-(k + 2 log2 N) fused into the last store.  The forward
pipeline (prescale -> forward -> undo) is timed too and reported beside it.

value  = whole-job round-trip Gpoints/s (sum over ranks; each rank owns a
         256-image shard: weak scaling, no collective on the data path);
e2e    = same, through the public API with pinned host buffers: every step
         copies the batch H2D, runs the pipeline and copies the result D2H;
roofline = the dominant kernel (the MX line pass, k_mx_lines: 4 launches per
         round trip) -- algorithmic HBM bytes (16 B per point per launch: one
         complex64 read + one write) / its CUDA-event duration per launch;
cpu_baseline = the C oracle (oracle/, a port of the reference algorithm)
         on a bounded sample of the same workload, all host threads.

`--impl reference` times that CPU port alone (rank 0; other ranks exit).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MX-FFT2 fwd+round-trip Gpoints/s; fraction of HBM roofline; PSNR delta vs oracle"
BYTES_PER_POINT = 16  # one complex64 read + one complex64 write per point per operation


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(PRESETS),
                    help="BASELINE.json configs[0..4] (c2 = configs[1], the headline)")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--fmt", default=None)
    ap.add_argument("--block", type=int, default=None)
    ap.add_argument("--noise", type=float, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the pipeline eagerly instead of replaying a captured CUDA graph")
    a = ap.parse_args()
    for key, v in PRESETS[a.config].items():
        if getattr(a, key) is None:
            setattr(a, key, v)
    return a


# BASELINE.json configs (per rank for c1-c4; c5 is one image split by rows)
PRESETS = {
    "c1": dict(batch=1, n=256, fmt="e4m3", block=32, noise=0.01),
    "c2": dict(batch=256, n=256, fmt="e4m3", block=32, noise=0.01),
    "c3": dict(batch=64, n=512, fmt="e3m2", block=32, noise=0.01),
    "c4": dict(batch=4096, n=128, fmt="e4m3", block=32, noise=0.05),
    "c5": dict(batch=1, n=16384, fmt="e4m3", block=32, noise=0.01),
}


def config_of(a, world):
    if a.config == "c5":
        return {
            "workload": f"C5: one {a.n}^2 complex64 synthetic k-space image, rows split over {world} "
                        f"GPU(s), {a.fmt.upper()} B={a.block}, global prescale + forward + inverse",
            "n": a.n, "format": a.fmt, "block_size": a.block, "noise": a.noise,
            "parallelism": f"row slabs x{world}, all-to-all transposes (NCCL)" if world > 1 else
                           "1 GPU: transposed-store row passes",
            "l2": "image (%.1f GB) far exceeds the 126 MB L2" % (a.n * a.n * 8 / 1e9),
        }
    return {
        "workload": f"{a.config.upper()}: {a.batch} x {a.n}^2 complex64 synthetic k-space per rank, "
                    f"{a.fmt.upper()} B={a.block}, prescale + forward + inverse (round trip)",
        "batch_per_rank": a.batch, "n": a.n, "format": a.fmt, "block_size": a.block,
        "noise": a.noise, "parallelism": f"batch-shard x{world} (no collective)",
        "l2": "inputs+outputs (2 x %.0f MB per rank) exceed the 126 MB L2" % (a.batch * a.n * a.n * 8 / 1e6),
    }


def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, dev_index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_baseline(x, fmt, block, seconds, threads=None):
    """Round-trip pipelines of the C oracle on whole images, all host threads,
    until `seconds` of wall time; returns Gpoints/s and the sample description."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor

    threads = threads or os.cpu_count() or 1
    n = x.shape[-1]
    plan = O.make_plan(n, O.ALL_MX[fmt], block)
    done = 0
    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        while True:
            idx = [(done + i) % x.shape[0] for i in range(threads)]
            list(ex.map(lambda i: O.pipeline(x[i], plan, True), idx))
            done += threads
            if time.perf_counter() - t0 >= seconds:
                break
    dt = time.perf_counter() - t0
    return done * n * n / dt / 1e9, threads, f"{done} round-trip pipelines of {n}^2 images ({dt:.1f} s)"


def run_reference(a, rank, world):
    if rank != 0:
        return
    if a.config == "c5":
        vals = []
        t0 = time.perf_counter()
        per_step = max(1.0, a.cpu_seconds / max(1, a.steps))
        for _ in range(a.steps):
            rate, cores, sample = cpu_rows_rate(a.n, a.fmt, a.block, per_step)
            vals.append(rate / 4 / 1e9)
        value = float(statistics.mean(vals))
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpoints/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": (time.perf_counter() - t0) / a.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 carry / fp8-e4m3 codes", "data": "synthetic", "config": config_of(a, world),
            "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": cores, "kind": "port",
                             "sample": f"per step: {sample}; round trip = 4 row passes"},
            "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }), flush=True)
        return
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    nimg = max(8, os.cpu_count() or 8)
    x = ellipse_kspace_batch(nimg, a.n, seed=0, noise=a.noise)
    per_step = max(1.0, a.cpu_seconds / max(1, a.steps))
    for _ in range(a.warmup):
        cpu_baseline(x, a.fmt, a.block, 0.0)
    vals = []
    t0 = time.perf_counter()
    for _ in range(a.steps):
        v, cores, sample = cpu_baseline(x, a.fmt, a.block, per_step)
        vals.append(v)
    total = time.perf_counter() - t0
    value = float(statistics.mean(vals))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpoints/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": total / a.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 carry / fp8-e4m3 codes", "data": "synthetic",
        "config": config_of(a, world),
        "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": cores, "kind": "port",
                         "sample": f"per step: {sample}"},
        "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_rows_rate(n, fmt, block, seconds, threads=None):
    """The oracle's row pass on seeded n-point rows, all host threads, for
    `seconds`; returns row-points per second (one pass)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from concurrent.futures import ThreadPoolExecutor

    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(0)
    rows = (rng.standard_normal((threads, 4, n)) + 1j * rng.standard_normal((threads, 4, n))).astype(np.complex64)
    plan = O.make_plan(n, O.ALL_MX[fmt], block)
    done, t0 = 0, time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        while True:
            list(ex.map(lambda i: O.fft_batch(rows[i], plan, False), range(threads)))
            done += threads * 4
            if time.perf_counter() - t0 >= seconds:
                break
    dt = time.perf_counter() - t0
    return done * n / dt, threads, f"{done} oracle row transforms of {n} points ({dt:.1f} s)"


def run_c5(a, rank, world, local):
    """C5: one n^2 image.  1 GPU: global prescale + fft2 with transposed-store
    passes.  N GPUs: row slabs, global prescale over all ranks, all-to-all
    transposes (paper_2512_04317_b200/distributed.py)."""
    import torch
    import torch.distributed as dist

    import paper_2512_04317_b200 as mx
    from paper_2512_04317_b200 import _native, distributed as D
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = D.Comm()
    n = a.n
    r0, r1 = D.shard_range(n, rank, world)
    x = ellipse_kspace_device(n, 7, noise=a.noise, rows=(r0, r1))
    plan = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(a.fmt), a.block))
    cfg = mx.PrescaleConfig()
    ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, 1)) if world == 1 else 1,
                     dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    kt = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def step(roundtrip=True, xin=None):
        xin = x if xin is None else xin
        res = D.compute_prescale_global(xin, cfg, comm)
        if world == 1:
            kt.fill_(res.k)
            return mx.fft2_device(xin[None], plan, "roundtrip" if roundtrip else "forward", k=kt,
                                  out=y[None], workspace=ws)
        return D.fft2_slab(xin, plan, "roundtrip" if roundtrip else "forward", comm, k=res.k)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        comm.sum_(torch.zeros(1, device="cuda"))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device="cuda")
        return float(comm.max_(ms).item())

    pts = n * n
    for _ in range(a.warmup):
        step()
    launches0 = _native.launch_count()
    with ClockSampler(local) as clk:
        ms = timed(step, a.steps, 0)
    launches = (_native.launch_count() - launches0) // max(1, a.steps)
    ms_fwd = timed(lambda: step(False), max(2, a.steps // 2), 1)
    # line pass (the dominant kernel): a plain forward fft2 on one GPU = 2 passes
    ms_pass = None
    if world == 1:
        ms_pass = timed(lambda: mx.fft2_device(x[None], plan, "forward", out=y[None], workspace=ws),
                        max(2, a.steps // 2), 1) / 2
    # e2e: pinned host slab in, result out, every step
    h_in = x.cpu().pin_memory()
    h_out = torch.empty(h_in.shape, dtype=h_in.dtype).pin_memory()
    xd = torch.empty_like(x)

    def e2e_step():
        xd.copy_(h_in, non_blocking=True)
        out = step(True, xd)
        h_out.copy_(out.reshape(h_out.shape), non_blocking=True)

    ms_e2e = timed(e2e_step, 2, 1)
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        rate, cores, sample = cpu_rows_rate(n, a.fmt, a.block, a.cpu_seconds)
        # a round trip is four row passes over the n^2 points
        cpu = {"value": rate / 4 / 1e9, "unit": "Gpoints/s", "cores": cores, "kind": "port",
               "sample": sample + "; round trip = 4 row passes of the image"}
    if rank == 0:
        peak, peak_src = measured_peak_hbm()
        value = pts / (ms * 1e-3) / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": "Gpoints/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 carry / fp8-e4m3 codes", "data": "synthetic",
            "config": config_of(a, world),
            "forward": {"value": pts / (ms_fwd * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": ms_fwd},
            "roofline": None if ms_pass is None else {
                "bound": "hbm", "kernel": "mx_line_pass (n=16384, k_mx_lines_big)",
                "achieved": BYTES_PER_POINT * pts / (ms_pass * 1e-3) / 1e9, "peak": peak,
                "peak_source": peak_src, "unit": "GB/s",
                "frac": BYTES_PER_POINT * pts / (ms_pass * 1e-3) / 1e9 / peak, "traffic": None,
                "kernel_ms": {"mx_line_pass": ms_pass}},
            "e2e": {"value": pts / (ms_e2e * 1e-3) / 1e9, "unit": "Gpoints/s",
                    "h2d_bytes_per_step": (r1 - r0) * n * 8 * world, "d2h_bytes_per_step": (r1 - r0) * n * 8 * world,
                    "ms_per_step": ms_e2e},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "parity": "tests/test_gpu_parity.py::test_c5_full_size_16384 (exact global prescale; rows and "
                      "columns equal to the oracle)",
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(a.gpus)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if a.config == "c5":
        run_c5(a, rank, world, local)
        return

    import torch
    import torch.distributed as dist

    import paper_2512_04317_b200 as mx
    from paper_2512_04317_b200 import _native
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    fmt = mx.get_mx_format(a.fmt)
    plan = mx.make_plan(a.n, mx.ModeSpec.mx(fmt, a.block))
    cfg = mx.PrescaleConfig()
    x_host = ellipse_kspace_batch(a.batch, a.n, seed=1000 * rank, noise=a.noise)
    x = torch.from_numpy(x_host).cuda()
    y = torch.empty_like(x)
    kbuf = torch.empty(a.batch, dtype=torch.int32, device="cuda")
    rbuf = torch.empty((a.batch, 40), dtype=torch.uint8, device="cuda")
    pts = a.batch * a.n * a.n
    stream = torch.cuda.current_stream()

    def step(roundtrip=True, xin=x):
        mx.pipeline_device(xin, plan, cfg, roundtrip=roundtrip, out=y, k=kbuf, res=rbuf)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return e0.elapsed_time(e1) / steps

    # ---- headline: round trip, device-resident ----
    # The step is captured once as a CUDA graph (same kernels, same buffers)
    # and replayed: no host launch gaps between its 7-8 dependent kernels.
    def graphed(fn):
        if a.no_graph:
            return fn, None
        for _ in range(2):  # plan tables, workspaces, kernel attributes: outside the capture
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        l0 = _native.launch_count()
        with torch.cuda.graph(g):
            fn()
        return g.replay, _native.launch_count() - l0

    run_rt, per_step = graphed(step)
    for _ in range(a.warmup):
        run_rt()
    launches0 = _native.launch_count()
    with ClockSampler(local) as clk:
        ms = timed(run_rt, a.steps, 0)
    launches = per_step * a.steps if per_step is not None else _native.launch_count() - launches0
    ms = max_over_ranks(ms)
    value = world * pts / (ms * 1e-3) / 1e9

    # ---- forward pipeline ----
    run_fwd, _ = graphed(lambda: step(False))
    ms_fwd = max_over_ranks(timed(run_fwd, a.steps, 2))
    fwd_value = world * pts / (ms_fwd * 1e-3) / 1e9

    # ---- per-kernel timing for the roofline (same stream, CUDA events) ----
    ms_stats = timed(lambda: mx.prescale_stats_device(x, a.batch, a.n * a.n, cfg, k_out=kbuf,
                                                      res_out=rbuf), a.steps, 2)
    # the line kernel as the pipeline runs it: a forward fft2 = two row passes
    # with transposed stores (scratch from torch's caching allocator)
    ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, a.batch)),
                     dtype=torch.uint8, device="cuda")
    ms_pass = timed(lambda: mx.fft2_device(x, plan, "forward", out=y, workspace=ws), a.steps, 2) / 2
    kernels = {"prescale_stats": ms_stats, "mx_line_pass": ms_pass}
    # share of the round-trip step: stats once, four line passes
    share = {"prescale_stats": ms_stats / ms, "mx_line_pass": 4 * ms_pass / ms}
    dom = "mx_line_pass"
    peak, peak_src = measured_peak_hbm()
    achieved = BYTES_PER_POINT * pts / (kernels[dom] * 1e-3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = (json.load(open(tr_path)).get(a.config) or {}).get(dom)
        except Exception:
            traffic = None

    # ---- e2e through the public API with pinned host buffers ----
    h_in = torch.from_numpy(x_host).pin_memory()
    h_out = torch.empty(h_in.shape, dtype=h_in.dtype).pin_memory()
    xd = torch.empty_like(x)

    def e2e_step():  # public host-buffer API: H2D / compute / D2H overlapped in slices
        mx.pipeline_host(h_in, plan, cfg, True, out_host=h_out, chunks=8)

    ms_e2e = max_over_ranks(timed(e2e_step, max(5, a.steps // 5), 2))
    e2e = world * pts / (ms_e2e * 1e-3) / 1e9

    # ---- parity spot check of the timed output (image 0) against the oracle ----
    step()
    torch.cuda.synchronize()
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    oplan = O.make_plan(a.n, O.ALL_MX[a.fmt], a.block)
    out_o, rss_o, k_o = O.pipeline(x_host[0], oplan, True)
    got = y[0].cpu().numpy().astype(np.complex128)
    bit_exact = bool(np.array_equal(got, out_o[0]))
    ref = np.abs(x_host[0].astype(np.complex128))
    psnr_delta = abs(O.psnr(ref, np.abs(got)) - O.psnr(ref, rss_o))

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        v, cores, sample = cpu_baseline(x_host[: max(8, os.cpu_count() or 8)], a.fmt, a.block,
                                        a.cpu_seconds)
        cpu = {"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Gpoints/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 carry / fp8-e4m3 codes",
            "data": "synthetic", "config": config_of(a, world),
            "hbm_fraction": value / world * BYTES_PER_POINT / peak,
            "forward": {"value": fwd_value, "unit": "Gpoints/s", "ms_per_step": ms_fwd,
                        "hbm_fraction": fwd_value / world * BYTES_PER_POINT / peak},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic,
                         "algorithmic_bytes_per_launch": BYTES_PER_POINT * pts,
                         "kernel_ms": kernels, "share_of_step": share},
            "e2e": {"value": e2e, "unit": "Gpoints/s", "h2d_bytes_per_step": pts * 8,
                    "d2h_bytes_per_step": pts * 8, "ms_per_step": ms_e2e},
            "gpu_launches": int(launches),
            "launch": "eager" if a.no_graph else "CUDA graph replay of the captured step",
            "clocks": clk.summary(),
            "parity": {"image0_bit_exact_vs_oracle": bit_exact, "k_oracle": k_o,
                       "k_gpu": int(kbuf[0].item()), "psnr_delta_db": psnr_delta},
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
