"""MX-FFT2 benchmark (BASELINE.json metric) on N GPUs of one node.

Headline workload: BASELINE.json configs[3] ("C4"), the largest single-GPU
configuration -- a batch of 4096 seeded synthetic k-space images, 128 x 128
complex64 each (ellipse phantoms + 5% complex Gaussian noise,
paper_2512_04317_b200/workloads.py), MXFP8 E4M3, B = 32, round trip.
One step = the round-trip pipeline over the whole batch on the GPU: per-image
prescale statistics (amax + tau-percentile selection, k on device) -> forward
MX-FFT2 with x*2^k fused into the first load -> inverse MX-FFT2 ->
x 2^-(k + 2 log2 N) fused into the last store.

Every other BASELINE configuration is measured in the same run and nested
under "configs" (C1; C2 E4M3 / E5M2; C3 E3M2 / E2M3 / E2M1 x B 16 / 32 / 64;
C4; C5), each with its own round-trip and forward rates, kernel times,
roofline fraction, a bit-exactness check of image 0 against the CPU oracle,
and a bounded CPU-oracle sample.

value  = whole-job round-trip Gpoints/s (sum over ranks; each rank owns a
         full per-rank batch: weak scaling, no collective on the data path);
e2e    = the same, through the public host-buffer API (pipeline_host) with
         pinned host buffers: every step copies the batch H2D, runs the
         pipeline and copies the result D2H;
roofline = the dominant kernel: algorithmic HBM bytes (16 B per point per
         launch: one complex64 read + one write) / its CUDA-event duration;
cpu_baseline = the C oracle (oracle/, a port of the reference algorithm)
         on a bounded sample of the same workload, all host threads.

`--impl reference` times that CPU port alone (rank 0; other ranks exit).
`--gpus N` without torchrun spawns the N ranks itself (127.0.0.1).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MX-FFT2 fwd+round-trip Gpoints/s; fraction of HBM roofline; PSNR delta vs oracle"
BYTES_PER_POINT = 16  # one complex64 read + one complex64 write per point per operation
L2_BYTES = 126 * 2**20

# BASELINE.json configs (batch per rank for C1-C4; C5 is one image split by rows)
CONFIGS = {
    "c1": dict(batch=1, n=256, fmt="e4m3", block=32, noise=0.01),
    "c2_e4m3": dict(batch=256, n=256, fmt="e4m3", block=32, noise=0.01),
    "c2_e5m2": dict(batch=256, n=256, fmt="e5m2", block=32, noise=0.01),
    **{f"c3_{f}_b{b}": dict(batch=64, n=512, fmt=f, block=b, noise=0.01)
       for f in ("e3m2", "e2m3", "e2m1") for b in (16, 32, 64)},
    "c4": dict(batch=4096, n=128, fmt="e4m3", block=32, noise=0.05),
    "c5": dict(batch=1, n=16384, fmt="e4m3", block=32, noise=0.01),
}
ALIASES = {"c2": "c2_e4m3", "c3": "c3_e3m2_b32"}
HEADLINE = "c4"
# configurations measured beside the headline when N > 1 (the sweep is N = 1)
MULTI_SWEEP = ("c2_e4m3", "c3_e2m1_b32", "c5")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS) + sorted(ALIASES),
                    help="the headline configuration (default: c4 = BASELINE configs[3])")
    ap.add_argument("--no-sweep", action="store_true", help="measure the headline only")
    ap.add_argument("--sweep-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sweep-cpu-seconds", type=float, default=1.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the pipeline eagerly instead of replaying a captured CUDA graph")
    a = ap.parse_args()
    a.config = ALIASES.get(a.config, a.config)
    return a


def describe(name, c, world):
    if name == "c5":
        return {
            "workload": f"C5: one {c['n']}^2 complex64 synthetic k-space image, rows split over {world} GPU(s), "
                        f"{c['fmt'].upper()} B={c['block']}, global prescale + forward + inverse",
            "n": c["n"], "format": c["fmt"], "block_size": c["block"], "noise": c["noise"],
            "parallelism": f"row slabs x{world}, all-to-all transposes (NCCL)" if world > 1 else
                           "1 GPU: row passes + tiled transposes",
            "l2": "image (%.1f GB) far exceeds the 126 MB L2" % (c["n"] ** 2 * 8 / 1e9),
        }
    ws = c["batch"] * c["n"] ** 2 * 8
    return {
        "workload": f"{name.upper()}: {c['batch']} x {c['n']}^2 complex64 synthetic k-space per rank, "
                    f"{c['fmt'].upper()} B={c['block']}, prescale + forward + inverse (round trip)",
        "batch_per_rank": c["batch"], "n": c["n"], "format": c["fmt"], "block_size": c["block"],
        "noise": c["noise"], "parallelism": f"batch-shard x{world} (no collective)",
        "l2": ("inputs+outputs (2 x %.0f MB per rank) exceed the 126 MB L2" % (ws / 1e6)) if 2 * ws > L2_BYTES
        else "working set fits in L2: a 256 MB buffer is written between timed steps (L2 flushed)",
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


# ---------------------------------------------------------------------------
# CPU legs (the oracle is the checker and the CPU baseline, never the product)
# ---------------------------------------------------------------------------
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O

    return O


def cpu_baseline(x, fmt, block, seconds, threads=None):
    """Round-trip pipelines of the C oracle on whole images, all host threads,
    until `seconds` of wall time; returns Gpoints/s, threads and the sample."""
    from concurrent.futures import ThreadPoolExecutor

    O = _oracle()
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


def cpu_rows_rate(n, fmt, block, seconds, threads=None):
    """The oracle's row pass on seeded n-point rows, all host threads, for
    `seconds`; returns row-points per second (one pass)."""
    from concurrent.futures import ThreadPoolExecutor

    O = _oracle()
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


def cpu_record(name, c, seconds):
    if name == "c5":
        rate, cores, sample = cpu_rows_rate(c["n"], c["fmt"], c["block"], seconds)
        return {"value": rate / 4 / 1e9, "unit": "Gpoints/s", "cores": cores, "kind": "port",
                "sample": sample + "; round trip = 4 row passes of the image"}
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    nimg = max(8, os.cpu_count() or 8)
    x = ellipse_kspace_batch(nimg, c["n"], seed=0, noise=c["noise"])
    v, cores, sample = cpu_baseline(x, c["fmt"], c["block"], seconds)
    return {"value": v, "unit": "Gpoints/s", "cores": cores, "kind": "port", "sample": sample}


def run_reference(a, rank, world):
    """The reference arm: the CPU port of the reference path on the headline
    config, all host threads, each step a bounded sample (rank 0 only)."""
    if rank != 0:
        return
    c = CONFIGS[a.config]
    per_step = max(1.0, a.cpu_seconds / max(1, a.steps))
    vals = []
    for _ in range(min(a.warmup, 1)):
        cpu_record(a.config, c, 0.5)
    t0 = time.perf_counter()
    last = None
    for _ in range(a.steps):
        last = cpu_record(a.config, c, per_step)
        vals.append(last["value"])
    total = time.perf_counter() - t0
    value = float(statistics.mean(vals))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpoints/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": total / a.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if a.config == "c5" else "weak", "vs_baseline": None,
        "dtype": "f32 carry / mx element codes", "data": "synthetic", "config": describe(a.config, c, world),
        "cpu_baseline": {"value": value, "unit": "Gpoints/s", "cores": last["cores"], "kind": "port",
                         "sample": "per step: " + last["sample"]},
        "e2e": {"value": value, "unit": "Gpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU legs
# ---------------------------------------------------------------------------
class Ctx:
    def __init__(self, rank, world, local):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.rank, self.world, self.local = rank, world, local
        self.stream = torch.cuda.current_stream()
        self._flush = None

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, v):
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def flush_l2(self):
        if self._flush is None:
            self._flush = self.torch.empty(256 << 20, dtype=self.torch.uint8, device="cuda")
        self._flush.fill_(1)

    def timed(self, fn, steps, warmup, flush=False):
        """Mean ms per call: CUDA events on the launching stream, a barrier and a
        synchronize on both sides, max over ranks.  flush: the working set fits
        in L2, so each call is timed alone after writing a 256 MB buffer."""
        torch = self.torch
        for _ in range(warmup):
            fn()
        self.barrier()
        torch.cuda.synchronize()
        if not flush:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            for _ in range(steps):
                fn()
            e1.record(self.stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
        else:
            evs = []
            for _ in range(steps):
                self.flush_l2()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(self.stream)
                fn()
                e1.record(self.stream)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in evs) / steps
        self.barrier()
        return self.max_over_ranks(ms)


_INPUTS = {}


def batch_input(c, rank):
    from paper_2512_04317_b200.workloads import ellipse_kspace_batch

    key = (c["batch"], c["n"], c["noise"], rank)
    if key not in _INPUTS:
        _INPUTS.clear()
        _INPUTS[key] = ellipse_kspace_batch(c["batch"], c["n"], seed=1000 * rank + c["n"], noise=c["noise"])
    return _INPUTS[key]


def measure_batch(ctx, name, c, steps, warmup, graph=True, e2e=False, cpu_seconds=0.0):
    """One batched configuration (C1-C4): round trip and forward pipelines,
    kernel times, roofline, image-0 parity against the oracle, CPU sample."""
    import paper_2512_04317_b200 as mx
    from paper_2512_04317_b200 import _native

    torch = ctx.torch
    world = ctx.world
    fmt = mx.get_mx_format(c["fmt"])
    plan = mx.make_plan(c["n"], mx.ModeSpec.mx(fmt, c["block"]))
    cfg = mx.PrescaleConfig()
    x_host = batch_input(c, ctx.rank)
    x = torch.from_numpy(x_host).cuda()
    y = torch.empty_like(x)
    kbuf = torch.empty(c["batch"], dtype=torch.int32, device="cuda")
    rbuf = torch.empty((c["batch"], 40), dtype=torch.uint8, device="cuda")
    pts = c["batch"] * c["n"] ** 2
    flush = 2 * pts * 8 <= 2 * L2_BYTES

    fused_ok = bool(mx.fused_pipeline_supported(plan))

    fold_ok = bool(mx.mri.folded_pipeline_supported(plan))

    def step(roundtrip=True, fused=None, fold=False):
        mx.pipeline_device(x, plan, cfg, roundtrip=roundtrip, out=y, k=kbuf, res=rbuf, fused=fused, fold=fold)

    def graphed(fn):
        if not graph:
            return fn, None
        for _ in range(2):  # plan tables, workspaces, kernel attributes: outside the capture
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        l0 = _native.launch_count()
        with torch.cuda.graph(g):
            fn()
        return g.replay, _native.launch_count() - l0

    # n = 128 (C4): the three implementations of the pipeline are timed -- the
    # all-in-one fused kernel (statistics in the one-image-per-CTA kernel), the
    # statistics kernel + the fused image transform, and the statistics kernel
    # + four line passes -- and the fastest one is the measured configuration
    L = _native.lib()
    alt = None
    fused, knob, fold = False, 1, False
    variants = {}
    if fused_ok:
        variants = {"fused_all_in_one": (True, 1, False), "stats_then_fused_fft2": (False, 1, False),
                    "stats_then_line_passes": (False, 0, False)}
    if fold_ok:
        # compute_prescale folded into the first line pass (mxfft_pipeline_folded)
        variants.setdefault("stats_then_line_passes", (False, 0 if fused_ok else 1, False))
        variants["statistics_folded_into_first_line_pass"] = (False, 0 if fused_ok else 1, True)
    if variants:
        t = {}
        for vname, (f, kn, fo) in variants.items():
            L.mxfft_fused_image(kn if fused_ok else -1)
            g_rt, _ = graphed(lambda f=f, fo=fo: step(True, f, fo))
            t[vname] = ctx.timed(g_rt, steps, warmup, flush)
        # the fastest variant, except that a line-pass variant (whose kernel's
        # HBM roofline is the per-pass one the other configurations report)
        # wins ties within 2 %: the fused transform is compute-bound and moves
        # 16 B per point per round trip, so its HBM fraction says nothing
        best = min(t, key=t.get)
        lp_best = min((v for v in t if v.endswith("line_passes") or v.endswith("line_pass")), key=t.get)
        if t[lp_best] <= 1.02 * t[best]:
            best = lp_best
        fused, knob, fold = variants[best]
        alt = {"ms_per_step": t, "chosen": best,
               "value": {v: world * pts / (ms_ * 1e-3) / 1e9 for v, ms_ in t.items()}}
    L.mxfft_fused_image(knob if fused_ok else -1)
    run_rt, per_step = graphed(lambda: step(True, fused, fold))
    for _ in range(warmup):
        run_rt()
    l0 = _native.launch_count()
    with ClockSampler(ctx.local) as clk:
        ms = ctx.timed(run_rt, steps, 0, flush)
    launches = per_step * steps if per_step is not None else _native.launch_count() - l0
    run_fwd, _ = graphed(lambda: step(False, fused, fold))
    ms_fwd = ctx.timed(run_fwd, steps, 2, flush)
    unsettled = None
    if fold:  # rows the folded statistics could not settle (pipeline_resolve would re-run them): none expected
        from paper_2512_04317_b200.prescale import decode_results

        unsettled = int((decode_results(rbuf)["flags"] & 4 != 0).sum())

    # the dominant kernel, as the pipeline runs it
    if fused:
        dom = "mx_fused_image (k_mx_image: statistics + 4 line passes in shared memory)"
        kernels = {"mx_fused_image": ms}
        ms_dom = ms
        share = {"mx_fused_image": 1.0}
    elif fused_ok and knob:
        ms_stats = ctx.timed(lambda: mx.prescale_stats_device(x, c["batch"], c["n"] ** 2, cfg, k_out=kbuf,
                                                              res_out=rbuf), steps, 2, flush)
        ms_img = ctx.timed(lambda: mx.fft2_device(x, plan, "roundtrip", k=kbuf, out=y), steps, 2, flush)
        dom = "mx_fused_image (k_mx_image: the 4-pass round trip in shared memory, k given)"
        kernels = {"prescale_stats": ms_stats, "mx_fused_image": ms_img}
        ms_dom = ms_img
        share = {"prescale_stats": ms_stats / ms, "mx_fused_image": ms_img / ms}
    else:
        ms_stats = ctx.timed(lambda: mx.prescale_stats_device(x, c["batch"], c["n"] ** 2, cfg, k_out=kbuf,
                                                              res_out=rbuf), steps, 2, flush)
        ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, c["batch"])),
                         dtype=torch.uint8, device="cuda")
        ms_pass = ctx.timed(lambda: mx.fft2_device(x, plan, "forward", out=y, workspace=ws), steps, 2, flush) / 2
        dom = "mx_line_pass (k_mx_lines_tma: TMA tile load + butterfly stages + TMA transposed store)" if c["n"] in (
            128, 256, 512) else "mx_line_pass (k_mx_lines)"
        kernels = {"prescale_stats": ms_stats, "mx_line_pass": ms_pass}
        ms_dom = ms_pass
        share = {"prescale_stats": ms_stats / ms, "mx_line_pass": 4 * ms_pass / ms}
        if fold:
            # the step is: accumulator memset + first pass with the statistics + resolve + 3 plain passes;
            # the standalone statistics kernel (timed above for reference) is NOT part of it
            kernels = {"mx_line_pass": ms_pass, "mx_first_pass_with_statistics": max(ms - 3 * ms_pass, 0.0),
                       "prescale_stats_standalone_not_in_step": ms_stats}
            share = {"mx_line_pass": 3 * ms_pass / ms, "mx_first_pass_with_statistics": max(ms - 3 * ms_pass, 0.0) / ms}
    peak, peak_src = measured_peak_hbm()
    achieved = BYTES_PER_POINT * pts / (ms_dom * 1e-3) / 1e9
    traffic = None
    try:
        traffic = (json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(name) or {}).get(
            "mx_fused_image" if (fused or (fused_ok and knob)) else "mx_line_pass")
    except Exception:
        pass

    # the pass's second roofline: instruction issue.  Executed warp
    # instructions per launch from the committed ncu captures; issue rate = SMs x 4 x SM clock
    issue = None
    try:
        winst = (json.load(open(os.path.join(ROOT, "profiles", "instructions.json"))).get(name) or {}).get(
            "mx_line_pass")
        if winst and not (fused or (fused_ok and knob)):
            props = torch.cuda.get_device_properties(ctx.local)
            rate = props.multi_processor_count * 4 * (clk.summary().get("sm_mhz") or 1965) * 1e6
            issue = {"warp_instructions_per_launch": winst, "issue_floor_ms": winst / rate * 1e3,
                     "frac_of_issue_rate": winst / rate * 1e3 / ms_dom,
                     "hbm_floor_ms": BYTES_PER_POINT * pts / (peak * 1e9) * 1e3}
    except Exception:
        pass

    rec = {
        "value": world * pts / (ms * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": ms,
        "hbm_fraction": pts / (ms * 1e-3) / 1e9 * BYTES_PER_POINT / peak,
        "forward": {"value": world * pts / (ms_fwd * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": ms_fwd,
                    "hbm_fraction": pts / (ms_fwd * 1e-3) / 1e9 * BYTES_PER_POINT / peak},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": BYTES_PER_POINT * pts, "kernel_ms": kernels,
                     "share_of_step": share, "issue": issue},
        "gpu_launches": int(launches),
        "launch": "eager" if not graph else "CUDA graph replay of the captured step",
        "clocks": clk.summary(),
        "config": describe(name, c, world),
        "l2_flushed_between_steps": flush,
        "implementations": alt,
        "unsettled_stacks": unsettled,
    }

    if e2e:
        h_in = torch.from_numpy(x_host).pin_memory()
        h_out = torch.empty(h_in.shape, dtype=h_in.dtype).pin_memory()
        ms_e2e = ctx.timed(lambda: mx.pipeline_host(h_in, plan, cfg, True, out_host=h_out, chunks=14),
                           max(5, steps // 5), 2)
        rec["e2e"] = {"value": world * pts / (ms_e2e * 1e-3) / 1e9, "unit": "Gpoints/s",
                      "h2d_bytes_per_step": world * pts * 8, "d2h_bytes_per_step": world * pts * 8,
                      "ms_per_step": ms_e2e}
        # the ceiling of this box's PCIe path for the same bytes: one pinned H2D and one pinned D2H
        # of the whole batch running concurrently on two streams (no kernels)
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

        def both():
            cur = torch.cuda.current_stream()
            s1.wait_stream(cur)
            s2.wait_stream(cur)
            with torch.cuda.stream(s1):
                x.copy_(h_in, non_blocking=True)
            with torch.cuda.stream(s2):
                h_out.copy_(y, non_blocking=True)
            cur.wait_stream(s1)
            cur.wait_stream(s2)

        ms_pcie = ctx.timed(both, 5, 2)
        rec["e2e"]["pcie_copies_only_ms"] = ms_pcie
        rec["e2e"]["pcie_gbytes_per_s_each_way"] = pts * 8 / (ms_pcie * 1e-3) / 1e9
        rec["e2e"]["fraction_of_copies_only"] = ms_pcie / ms_e2e
        x.copy_(h_in)  # (restore the device input for the checks below)

    # parity spot check of the timed output (image 0) against the oracle
    step(True, fused)
    L.mxfft_fused_image(-1)
    torch.cuda.synchronize()
    O = _oracle()
    oplan = O.make_plan(c["n"], O.ALL_MX[c["fmt"]], c["block"])
    out_o, rss_o, k_o = O.pipeline(x_host[0], oplan, True)
    got = y[0].cpu().numpy().astype(np.complex128)
    ref = np.abs(x_host[0].astype(np.complex128))
    rec["parity"] = {"image0_bit_exact_vs_oracle": bool(np.array_equal(got, out_o[0])), "k_oracle": int(k_o),
                     "k_gpu": int(kbuf[0].item()),
                     "psnr_delta_db": abs(O.psnr(ref, np.abs(got)) - O.psnr(ref, rss_o))}
    if cpu_seconds > 0 and ctx.rank == 0 and world == 1:
        rec["cpu_baseline"] = cpu_record(name, c, cpu_seconds)
    return rec


def measure_c5(ctx, c, steps, warmup, e2e=False, cpu_seconds=0.0):
    """C5: one n^2 image.  1 GPU: global prescale + fft2 (row passes and tiled
    transposes), or the prescale folded into the first split pass.  N GPUs:
    row slabs, the global prescale folded into the first row pass (evidence
    combined with two small all-reduces), all-to-all transposes
    (paper_2512_04317_b200/distributed.py)."""
    import paper_2512_04317_b200 as mx
    from paper_2512_04317_b200 import _native, distributed as D
    from paper_2512_04317_b200.workloads import ellipse_kspace_device

    torch = ctx.torch
    world = ctx.world
    comm = D.Comm()
    n = c["n"]
    r0, r1 = D.shard_range(n, ctx.rank, world)
    x = ellipse_kspace_device(n, 7, noise=c["noise"], rows=(r0, r1))
    plan = mx.make_plan(n, mx.ModeSpec.mx(mx.get_mx_format(c["fmt"]), c["block"]))
    cfg = mx.PrescaleConfig()
    ws = torch.empty(int(_native.lib().mxfft_fft2_workspace_bytes(plan.handle, 1)) if world == 1 else 1,
                     dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    kt = torch.zeros(1, dtype=torch.int32, device="cuda")

    def step(roundtrip=True, xin=None):
        xin = x if xin is None else xin
        if world == 1:
            res = D.compute_prescale_global(xin, cfg, comm)
            kt.fill_(res.k)
            return mx.fft2_device(xin[None], plan, "roundtrip" if roundtrip else "forward", k=kt,
                                  out=y[None], workspace=ws)
        # N GPUs: the prescale rides on the first row pass of the slabs (two small all-reduces, one
        # read-back of k); 3 all-to-alls per round trip, the result stays as column slabs
        return D.pipeline_slab(xin, plan, cfg, roundtrip, comm, restore=False)[0]

    pts = n * n
    # 1 GPU: the global prescale can also ride on the first row pass (mxfft_pipeline_folded: no
    # statistics pass over x, no host synchronisation); both variants are timed, the faster one
    # is the measured configuration
    alt, unsettled = None, None
    step_std = step
    if world == 1 and mx.mri.folded_pipeline_supported(plan):
        rbuf = torch.empty((1, 40), dtype=torch.uint8, device="cuda")

        def step_fold(roundtrip=True, xin=None):
            xin = x if xin is None else xin
            return mx.pipeline_device(xin[None], plan, cfg, roundtrip, out=y[None], k=kt, res=rbuf)[0][0]

        t = {"global_statistics_then_fft2": ctx.timed(step_std, max(2, steps // 2), 2),
             "statistics_folded_into_first_row_pass": ctx.timed(step_fold, max(2, steps // 2), 2)}
        from paper_2512_04317_b200.prescale import decode_results

        unsettled = int((decode_results(rbuf)["flags"] & 4 != 0).sum())
        best = min(t, key=t.get)
        if unsettled:  # (not for this workload: the fold then needs the resolve's re-run)
            best = "global_statistics_then_fft2"
        if best != "global_statistics_then_fft2":
            step = step_fold
        alt = {"ms_per_step": t, "chosen": best, "value": {v: pts / (m_ * 1e-3) / 1e9 for v, m_ in t.items()}}
    for _ in range(warmup):
        step()
    l0 = _native.launch_count()
    with ClockSampler(ctx.local) as clk:
        ms = ctx.timed(step, steps, 0)
    launches = (_native.launch_count() - l0) // max(1, steps)
    ms_fwd = ctx.timed(lambda: step(False), max(2, steps // 2), 1)
    ms_pass = None
    if world == 1:  # the dominant kernel: a plain forward fft2 = 2 row passes + 2 transposes
        ms_fft2 = ctx.timed(lambda: mx.fft2_device(x[None], plan, "forward", out=y[None], workspace=ws),
                            max(2, steps // 2), 1)
        ms_rows = ctx.timed(lambda: mx.fft_rows_device(x, plan, False, out=y), max(2, steps // 2), 1)
        ms_pass = ms_rows
    peak, peak_src = measured_peak_hbm()
    rec = {
        "value": pts / (ms * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": ms, "scaling": "strong",
        "hbm_fraction": pts / (ms * 1e-3) / 1e9 * BYTES_PER_POINT / peak / world,
        "forward": {"value": pts / (ms_fwd * 1e-3) / 1e9, "unit": "Gpoints/s", "ms_per_step": ms_fwd},
        "roofline": None if ms_pass is None else {
            "bound": "hbm", "kernel": "mx_line_pass (n=16384 rows, k_mx_lines_big)",
            "achieved": BYTES_PER_POINT * pts / (ms_pass * 1e-3) / 1e9, "peak": peak, "peak_source": peak_src,
            "unit": "GB/s", "frac": BYTES_PER_POINT * pts / (ms_pass * 1e-3) / 1e9 / peak, "traffic": None,
            "kernel_ms": {"mx_line_pass": ms_pass, "fft2_forward": ms_fft2}},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "config": describe("c5", c, world),
        "exchange": None if world == 1 else "3 all-to-alls per round trip (output left as column slabs)",
        "implementations": alt,
        "unsettled_stacks": unsettled,
        "parity": "tests/test_gpu_r2.py::test_c5_full_size_roundtrip_vs_oracle (16384^2 forward and round "
                  "trip bit-exact vs the threaded oracle; exact global prescale)",
    }
    if e2e:
        h_in = x.cpu().pin_memory()
        h_out = torch.empty(h_in.shape, dtype=h_in.dtype).pin_memory()
        xd = torch.empty_like(x)

        def e2e_step():
            xd.copy_(h_in, non_blocking=True)
            out = step(True, xd)
            h_out.copy_(out.reshape(h_out.shape), non_blocking=True)

        ms_e2e = ctx.timed(e2e_step, 2, 1)
        rec["e2e"] = {"value": pts / (ms_e2e * 1e-3) / 1e9, "unit": "Gpoints/s",
                      "h2d_bytes_per_step": pts * 8, "d2h_bytes_per_step": pts * 8, "ms_per_step": ms_e2e}
    if cpu_seconds > 0 and ctx.rank == 0 and world == 1:
        rec["cpu_baseline"] = cpu_record("c5", c, cpu_seconds)
    return rec


def measure(ctx, name, steps, warmup, graph, e2e, cpu_seconds):
    c = CONFIGS[name]
    if name == "c5":
        return measure_c5(ctx, c, steps, warmup, e2e, cpu_seconds)
    return measure_batch(ctx, name, c, steps, warmup, graph, e2e, cpu_seconds)


def run_gpu(a, rank, world, local):
    import torch
    import torch.distributed as dist

    if local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs GPU {local}, but only {torch.cuda.device_count()} "
                         f"visible (--gpus {world} runs one process per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Ctx(rank, world, local)
    cpu_s = 0.0 if a.no_cpu_baseline else a.cpu_seconds
    head = measure(ctx, a.config, a.steps, a.warmup, not a.no_graph, not a.no_e2e, cpu_s)
    configs = {}
    if not a.no_sweep:
        names = [n for n in CONFIGS if n != a.config] if world == 1 else [n for n in MULTI_SWEEP if n != a.config]
        for name in names:
            try:
                configs[name] = measure(ctx, name, min(a.steps, a.sweep_steps), 2, not a.no_graph, False,
                                        0.0 if a.no_cpu_baseline else a.sweep_cpu_seconds)
            except Exception as e:  # one configuration failing must not hide the others
                configs[name] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.empty_cache()
    configs[a.config] = {k: v for k, v in head.items() if k != "e2e"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "Gpoints/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": head["ms_per_step"], "higher_is_better": True,
            "scaling": head.get("scaling", "weak"), "vs_baseline": None,
            "dtype": "f32 carry / mx element codes", "data": "synthetic (seeded ellipse phantoms + noise)",
            "config": head["config"], "headline": a.config,
            "hbm_fraction": head["hbm_fraction"], "forward": head["forward"], "roofline": head["roofline"],
            "e2e": head.get("e2e"), "gpu_launches": head["gpu_launches"], "launch": head.get("launch"),
            "clocks": head["clocks"], "parity": head["parity"], "cpu_baseline": head.get("cpu_baseline"),
            "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawned(local, world, port, argv):
    os.environ.update({"RANK": str(local), "LOCAL_RANK": str(local), "WORLD_SIZE": str(world),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.argv = argv
    main()


def main():
    a = parse()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        if a.impl == "reference":  # the reference arm runs on rank 0 only: no ranks to spawn
            run_reference(a, 0, a.gpus)
            return
        import torch.multiprocessing as mp

        mp.start_processes(_spawned, args=(a.gpus, _free_port(), list(sys.argv)), nprocs=a.gpus,
                           start_method="spawn")
        return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    run_gpu(a, rank, world, local)


if __name__ == "__main__":
    main()
