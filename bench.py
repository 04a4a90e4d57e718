#!/usr/bin/env python
"""Benchmark: 2D ATSFFT transforms/s at N=4096, k=100 (BASELINE.json metric).

Workload (BASELINE.json configs[2], "c3"): one 4096 x 4096 complex64 image per
rank per step whose spectrum has k=100 unit-magnitude random-phase coefficients
at distinct uniform positions plus complex Gaussian noise at 20 dB SNR
(seeded synthetic input, paper_1908_02461_b200.signals.sparse_image; the
reference ships no dataset).  A step is one full ``atsfft2d`` (TunerConfig()
defaults, est_loops=8): the adaptive tuning passes, the vote histogram, the
estimation loops, median, top-k and prune.

Legs printed on ONE JSON line (rank 0):
  value     transforms/s with the images resident in HBM: --steps transforms
            per rank, --concurrency of them in flight (distinct c3 images, one
            CUDA stream + native context per in-flight transform), CUDA events
            on the launch stream around the whole run (barrier + sync both
            sides, max over ranks).  The 134 MB images and the ~1 GB
            per-transform working set exceed the 126 MB L2, so no flush.
  latency   the same steps with one transform in flight (per-transform time).
  e2e       the value leg through the public API with the images in pinned
            HOST memory: every step's host->device copy and result download
            are inside the timed region.
  roofline  dominant kernel: algorithmic bytes per launch / CUDA-event launch
            time from the library's per-launch profiler (a separate
            instrumented pass over the same steps), against MEASURED_PEAKS.json.
  cpu_baseline  the numpy oracle port (oracle/sfft_oracle.py, pocketfft FFTs)
            on one full c3 transform on one host core (rank 0, N=1).
``--impl reference`` times that oracle port instead (the reference is a pure
Python package that cannot travel to the GPU box; oracle/ restates it), on all
host cores via a process pool, and prints the same line with impl=reference.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "2D ATSFFT transforms/sec at N=4096,k=100; achieved HBM GB/s vs B200 peak"
UNIT = "transforms/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--snr", type=float, default=20.0)
    ap.add_argument("--est-loops", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=3)
    ap.add_argument("--c4-images", type=int, default=96,
                    help="images in the batched (c4) throughput sample; 0 skips it")
    ap.add_argument("--concurrency", type=int, default=6)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(args, rank, j=0):
    """c3 image j of this rank (distinct seeds: 7 + rank + 1000 j)."""
    from paper_1908_02461_b200.signals import sparse_image
    return sparse_image(args.n, args.k, 7 + rank + 1000 * j, snr_db=args.snr)


def c4_image(i: int):
    """BASELINE configs[3] item i: 1024^2 c64, own seed, k ~ U[20, 200],
    log-uniform magnitudes in [0.1, 10], random phase, 25 dB SNR."""
    from paper_1908_02461_b200.signals import sparse_image
    seed = 100_000 + i
    k = int(np.random.default_rng(seed).integers(20, 201))
    return sparse_image(1024, k, seed, snr_db=25.0, magnitude="loguniform").x


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed
    region: an NVML thread every 10 ms (so even a short region gets samples),
    else `nvidia-smi -lms 100`."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = self.thread = None
        self.sm, self.smax, self.reasons = [], 0.0, set()

    def start(self):
        self.sm, self.smax, self.reasons = [], 0.0, set()
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {k: getattr(nv, v) for k, v in self.REASONS.items() if hasattr(nv, v)}
            self.stop_evt = threading.Event()

            def run():
                while True:
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.reasons.update(k for k, b in bits.items() if r & b)
                    if self.stop_evt.wait(0.01):
                        return

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001 - no NVML: fall back to nvidia-smi
            self.thread = None
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.dev)], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict | None:
        src = "nvml"
        if self.thread is not None:
            self.stop_evt.set()
            self.thread.join()
        elif self.proc is not None:
            src = "nvidia-smi"
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in open(self.path):
                f = [v.strip() for v in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    self.sm.append(float(f[1]))
                    self.smax = max(self.smax, float(f[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, f[5:9]):
                    if v.lower().startswith("active"):
                        self.reasons.add(nm)
            os.unlink(self.path)
        if not self.sm:
            return None
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": src}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def kernel_traffic():
    path = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def cpu_baseline(x, args):
    from oracle import sfft_oracle as O
    O.FAST = True
    t0 = time.perf_counter()
    O.atsfft(x, O.TunerParams(), args.est_loops, 11)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"one full ATSFFT transform of the c3 image ({args.n}^2 c64, k={args.k}, "
                      f"{args.snr:g} dB, est_loops={args.est_loops}) by the numpy oracle port "
                      f"(pocketfft FFTs), 1 thread, {dt:.1f} s"}


# ---------------------------------------------------------------- reference arm
def _ref_worker(args_tuple):
    import numpy as np  # noqa: F811
    from oracle import sfft_oracle as O
    O.FAST = True
    x, est_loops, seed = args_tuple
    t0 = time.perf_counter()
    O.atsfft(x, O.TunerParams(), est_loops, seed)
    return time.perf_counter() - t0


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp
    img = workload(args, 0)
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, 16))
    steps = max(1, min(args.steps, 2))
    warm = 1 if args.warmup > 0 else 0
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for _ in range(warm):
            pool.map(_ref_worker, [(img.x, args.est_loops, 11)] * procs)
        t0 = time.perf_counter()
        for _ in range(steps):
            pool.map(_ref_worker, [(img.x, args.est_loops, 11)] * procs)
        dt = time.perf_counter() - t0
    value = steps * procs / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "requested_steps": args.steps, "warmup": warm,
        "ms_per_step": dt / steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"c3: ATSFFT {args.n}x{args.n} c64, k={args.k}, {args.snr:g} dB, "
                               f"est_loops={args.est_loops}", "parallelism": f"{procs} host processes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "sample": f"{steps} step(s) x {procs} concurrent full c3 transforms of the "
                                   f"numpy oracle port (pocketfft FFTs), one per process"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://", world_size=world, rank=rank)
    dev = torch.device("cuda", local)
    import paper_1908_02461_b200 as P
    from paper_1908_02461_b200 import _native

    conc = max(1, args.concurrency)
    imgs = [workload(args, rank, j) for j in range(conc)]
    img = imgs[0]
    xs_dev = [torch.from_numpy(im.x).to(dev) for im in imgs]
    x_dev = xs_dev[0]
    cfg = P.TunerConfig()
    ctx = _native.context(local)
    stream = torch.cuda.current_stream(dev)
    from paper_1908_02461_b200 import batch as PB

    def step(x):
        return P.atsfft2d_arrays(x, cfg, args.est_loops, 11, precision=args.precision)

    def run_steps(items, fn, concurrency):
        """fn(item) for every item, `concurrency` in flight (one stream and
        native context per worker); returns the summed kernel launches."""
        def one(i):
            fn(items[i])
            return _native.context(local).last_launches
        return sum(PB._run(one, len(items), concurrency, dev))

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    # warm-up (also builds tables / workspace in every worker context): every
    # worker thread runs every distinct image once, then the usual warm-up steps
    for _ in range(max(args.warmup, 1)):
        (ij, vals), state = step(x_dev)
    for j in range(conc):
        PB.warm_workers(lambda j=j: step(xs_dev[j]), conc, dev)
    run_steps([xs_dev[i % conc] for i in range(max(args.warmup, 2 * conc))], step, conc)
    torch.cuda.synchronize()
    parity = None
    gold = os.path.join(ROOT, "tests", "golden", "c3_ats.npz")
    if rank == 0 and args.n == 4096 and args.k == 100 and args.snr == 20.0 and os.path.exists(gold):
        g = np.load(gold)
        ref = {tuple(c) for c in g["coords"].tolist()}
        got = [(b, c) for b, c, _ in state.history]
        ref_h = [(int(b), int(c)) for b, c in g["hist"][:, :2]]
        same_b = [b for b, _ in got] == [b for b, _ in ref_h]
        rel = max((abs(c1 - c2) / max(c2, 1) for (_, c1), (_, c2) in zip(got, ref_h)), default=0.0)
        parity = {"support_equal_to_reference": ref == {tuple(c) for c in ij.tolist()},
                  "coefficients": int(len(ij)),
                  "b_trajectory_equal": same_b,
                  "maxima_counts_max_rel_diff": rel,
                  "trajectory_within_tolerance": same_b and (rel <= 1e-4 if args.precision == "fp32"
                                                             else rel == 0.0)}

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)

    def timed(items, fn, concurrency):
        gc.collect()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        n_launch = run_steps(items, fn, concurrency)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), n_launch

    # the cyclic garbage collector stays off for the timed legs: a collection
    # pause (tens of ms over the run's Python objects) inside a ~15 ms region
    # would halve that sample; it is re-enabled before the CPU baseline
    gc.disable()
    if os.environ.get("SFFT2D_TRACE_ALLOC"):
        print("---- timed region", file=sys.stderr, flush=True)
    # ---- timed region: value (images resident in HBM, `conc` in flight)
    vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    sampler = ClockSampler(int(vis[local]) if len(vis) > local and vis[local].isdigit() else local)
    sampler.start()
    ms_max, launches = timed([xs_dev[i % conc] for i in range(args.steps)], step, conc)
    clocks = sampler.stop()
    value = world * args.steps / (ms_max / 1e3)

    if os.environ.get("SFFT2D_TRACE_ALLOC"):
        print("---- end of timed region", file=sys.stderr, flush=True)
    # ---- single-transform latency: one in flight, same steps
    lat_ms, _ = timed([x_dev] * args.steps, step, 1)
    latency = {"ms_per_transform": lat_ms / args.steps, "transforms_per_s": world * args.steps / (lat_ms / 1e3),
               "in_flight": 1}

    # ---- e2e: pinned host images, H2D + result D2H inside the region
    e2e = None
    if not args.no_e2e:
        hosts = []
        for im in imgs:
            h = torch.empty((args.n, args.n), dtype=torch.complex64, pin_memory=True)
            h.copy_(torch.from_numpy(im.x))
            hosts.append(h.numpy())
        d2h = [0]

        def step_host(xh):
            out, _st = P.atsfft2d(xh, cfg, args.est_loops, 11, precision=args.precision)
            d2h[0] += len(out) * (16 + (16 if args.precision == "fp64" else 8))

        run_steps(hosts, step_host, conc)
        d2h[0] = 0
        e2e_ms, _ = timed([hosts[i % conc] for i in range(args.steps)], step_host, conc)
        nperm = cfg.iters(args.n) + 2 + args.est_loops
        e2e = {"value": world * args.steps / (e2e_ms / 1e3), "unit": UNIT, "in_flight": conc,
               "h2d_bytes_per_step": args.n * args.n * 8 + nperm * 48,
               "d2h_bytes_per_step": d2h[0] // max(args.steps, 1)}

    # ---- batched throughput (c4 sample): independent 1024^2 images, resident
    # in HBM, `--concurrency` transforms in flight on separate streams
    batched = None
    if args.c4_images > 0:
        xs = [torch.from_numpy(c4_image(rank * args.c4_images + i)).to(dev)
              for i in range(args.c4_images)]
        seeds = [1 + i for i in range(args.c4_images)]
        for _ in range(3):   # every worker meets most images (workspace sizes settle)
            P.atsfft2d_batch(xs, cfg, args.est_loops, seeds, concurrency=args.concurrency,
                             precision=args.precision, arrays=True)
        torch.cuda.synchronize()
        samples = []
        bsampler = ClockSampler(sampler.dev)
        bsampler.start()
        for _ in range(3):
            gc.collect()
            barrier()
            torch.cuda.synchronize()
            e0.record(stream)
            P.atsfft2d_batch(xs, cfg, args.est_loops, seeds, concurrency=args.concurrency,
                             precision=args.precision, arrays=True)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            samples.append(world * args.c4_images / (float(t.item()) / 1e3))
        bclocks = bsampler.stop()
        batched = {"workload": f"c4 sample: {args.c4_images} independent 1024x1024 c64 images per "
                               "rank, k~U[20,200], log-uniform magnitudes, 25 dB, est_loops="
                               f"{args.est_loops}", "concurrency": args.concurrency,
                   "value": float(np.median(samples)), "samples": samples, "unit": UNIT,
                   "clocks": bclocks}
        del xs

    # ---- kernel-level roofline (instrumented pass, same workload)
    ctx.set_profiling(True)
    nprof = max(1, min(args.profile_steps, args.steps))
    pe0 = torch.cuda.Event(enable_timing=True)
    pe1 = torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for _ in range(nprof):
        step(x_dev)
    pe1.record(stream)
    torch.cuda.synchronize()
    rep = ctx.profile_report()
    ctx.set_profiling(False)
    prof_ms = pe0.elapsed_time(pe1)
    peak, peak_kind = peaks()
    top = max(rep.items(), key=lambda kv: kv[1][1]) if rep else None
    roofline = None
    if top:
        name, (cnt, tms, tbytes) = top
        achieved = (tbytes / cnt) / (tms / cnt / 1e3) / 1e9
        traffic = kernel_traffic().get(name)
        roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "alg_bytes_per_launch": tbytes / cnt,
                    "launches_per_step": cnt / nprof, "avg_launch_us": tms / cnt * 1e3,
                    "share_of_step": tms / prof_ms}
    kernels = {k: {"launches_per_step": v[0] / nprof, "ms_per_step": v[1] / nprof,
                   "GBps": (v[2] / v[1] / 1e6) if v[1] > 0 else None}
               for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])[:8]}

    # ---- dense cuFFT of the same image, for context only
    torch.cuda.synchronize()
    xc = x_dev.to(torch.complex64)
    for _ in range(3):
        torch.fft.fft2(xc)
    c0 = torch.cuda.Event(enable_timing=True)
    c1 = torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for _ in range(10):
        torch.fft.fft2(xc)
    c1.record(stream)
    torch.cuda.synchronize()
    cufft_ms = c0.elapsed_time(c1) / 10

    gc.enable()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(img.x, args)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": f"c3: ATSFFT {args.n}x{args.n} complex64, k={args.k}, "
                                   f"{args.snr:g} dB SNR, TunerConfig() defaults, est_loops="
                                   f"{args.est_loops}, one transform per rank per step, {conc} "
                                   f"distinct images, {conc} transforms in flight (one CUDA "
                                   f"stream each)",
                       "precision": args.precision, "l2": "inputs larger than L2 (134 MB image)",
                       "parallelism": f"independent transforms, {world} rank(s)"},
            "e2e": e2e, "latency": latency, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches, "kernels": kernels, "batched": batched,
            "context": {"cufft_dense_fft2_c64_ms": cufft_ms,
                        "detected_k": state.detected_k, "passes": state.passes,
                        "trajectory": [b for b, _, _ in state.history]},
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
