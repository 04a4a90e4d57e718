#!/usr/bin/env python
"""Benchmark: 2D ATSFFT transforms/s at N=4096, k=100 (BASELINE.json metric).

Headline workload (BASELINE.json configs[2], "c3"): one 4096 x 4096 complex64
image per rank per step whose spectrum has k=100 unit-magnitude random-phase
coefficients at distinct uniform positions plus complex Gaussian noise at
20 dB SNR (seeded synthetic input, ``signals.sparse_image``; the reference
ships no dataset).  A step is one full ``atsfft2d`` (TunerConfig() defaults,
est_loops=8): the adaptive tuning passes, the votes, the estimation loops,
median, top-k and prune.

One JSON line (rank 0) carries:
  value      c3 transforms/s with the images resident in HBM, --concurrency
             distinct images in flight (one CUDA stream + native context each),
             CUDA events around the whole run (barrier + sync both sides, max
             over ranks).  At N > 1 every rank runs its own transforms
             (replicas: the tuner passes are strictly sequential).
  latency    the same steps one at a time (per-transform time).
  e2e        the value leg through the public API with the images in pinned
             HOST memory: H2D of each image and the result D2H inside the
             timed region.
  roofline   dominant kernel (library per-launch CUDA events, algorithmic bytes
             per DESIGN §3) against MEASURED_PEAKS.json, plus a transform-level
             figure (all kernels' algorithmic bytes per transform / time).
  legs       every other BASELINE config, each with its own parity check:
             c3_fp64 (verification precision), c1 (SFFT known k, 256^2 c128),
             c2 (ATSFFT 1024^2), c4 (2048 images sharded over the ranks,
             strong scaling), c5 (16384^2, k in {64, 256, 1024, 4096}, the
             estimation loops split over the ranks), c3_sfft (known-k SFFT,
             location + estimation loops split over the ranks).
  cpu_baseline  the numpy oracle port on one host core, one c3 transform.

``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` with N ranks (one per GPU, NCCL).
``--impl reference`` times the reference's CPU path instead (rank 0 only):
the oracle port on all host cores (``value``) and, when ``baseline/_ref``
holds the unmodified reference package, that package on c1, c2 and c3.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import socket
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
ALL_LEGS = ("c3_fp64", "c1", "c2", "c4", "c5", "c3_sfft")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["fp32", "fp64"], default="fp32")
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--snr", type=float, default=20.0)
    ap.add_argument("--est-loops", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=10)
    ap.add_argument("--legs", default=",".join(ALL_LEGS),
                    help=f"comma list of extra legs ({','.join(ALL_LEGS)}), or 'none'")
    ap.add_argument("--c4-images", type=int, default=2048)
    ap.add_argument("--c5-ks", default="64,256,1024,4096")
    ap.add_argument("--concurrency", type=int, default=6)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn(args) -> int:
    """--gpus N outside torchrun: re-launch under torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def workload(args, rank, j=0):
    """c3 image j of this rank (distinct seeds: 7 + rank + 1000 j)."""
    from paper_1908_02461_b200.signals import sparse_image
    return sparse_image(args.n, args.k, 7 + rank + 1000 * j, snr_db=args.snr)


def c4_params(i: int):
    """BASELINE configs[3] item i: 1024^2 c64, own seed, k ~ U[20, 200],
    log-uniform magnitudes in [0.1, 10], random phase, 25 dB SNR
    (oracle/make_golden.py c4_bench_image is the same definition)."""
    seed = 100_000 + i
    k = int(np.random.default_rng(seed).integers(20, 201))
    return seed, k


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


def kernel_traffic(config_key: str) -> dict:
    """ncu DRAM bytes per launch by kernel, for one (config, precision) key,
    from profiles/kernel_traffic.json (written from an ncu --set full capture
    of that exact configuration; a kernel or configuration without a capture
    reports null)."""
    path = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(config_key, {})
    except (OSError, ValueError):
        return {}


def golden(name):
    path = os.path.join(ROOT, "tests", "golden", f"{name}.npz")
    return dict(np.load(path)) if os.path.exists(path) else None


def compare(out_ij, out_v, g, precision, state=None):
    """Support / value / trajectory parity of one transform against a
    reference golden (tolerances of tests/test_gpu_parity.py)."""
    tol = 1e-10 if precision == "fp64" else 1e-4
    ref = dict(zip(map(tuple, g["coords"].tolist()), g["vals"]))
    got = dict(zip(map(tuple, np.asarray(out_ij).tolist()), np.asarray(out_v)))
    same = set(got) == set(ref)
    worst = 0.0
    if same and ref:
        vmax = max(abs(v) for v in ref.values())
        worst = max(abs(got[k] - v) / max(abs(v), 1e-3 * vmax) for k, v in ref.items())
    res = {"support_equal": same, "coefficients": len(got), "max_rel_err": float(worst),
           "within_tolerance": bool(same and worst <= tol), "tolerance": tol}
    if state is not None and "hist" in g:
        b_got = [b for b, _, _ in state.history]
        b_ref = [int(b) for b in g["hist"][:, 0]]
        res["b_trajectory_equal"] = b_got == b_ref
        if precision == "fp64":
            c_got = [c for _, c, _ in state.history]
            res["counts_equal"] = c_got == [int(c) for c in g["hist"][:, 1]]
        res["within_tolerance"] = res["within_tolerance"] and res["b_trajectory_equal"]
    return res


class Bench:
    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.args = args
        self.torch, self.dist = torch, dist
        self.world, self.rank, self.local = dist_env()
        # SFFT2D_BENCH_SAME_DEVICE=1: every rank on cuda:0 with gloo — a
        # plumbing check of the N > 1 path on a one-GPU box (the ranks' kernels
        # never wait on one another; the numbers are not a scaling measurement)
        self.same = os.environ.get("SFFT2D_BENCH_SAME_DEVICE") == "1"
        if self.same:
            self.local = 0
        torch.cuda.set_device(self.local)
        if self.world > 1:
            if self.same:
                dist.init_process_group("gloo", init_method="env://", world_size=self.world,
                                        rank=self.rank)
            else:
                dist.init_process_group("nccl", init_method="env://", world_size=self.world,
                                        rank=self.rank, device_id=torch.device("cuda", self.local))
        self.dev = torch.device("cuda", self.local)
        self.stream = torch.cuda.current_stream(self.dev)
        vis = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
        self.nvml_index = int(vis[self.local]) if len(vis) > self.local and vis[self.local].isdigit() \
            else self.local

    def barrier(self):
        if self.world > 1:
            if self.same:
                self.dist.barrier()
            else:
                self.dist.barrier(device_ids=[self.local])

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64,
                              device="cpu" if self.same else self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, fn):
        """ms of fn() on the device (barrier + sync both sides, CUDA events on
        the current stream, max over ranks) and fn's return value."""
        torch = self.torch
        gc.collect()
        self.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(self.stream)
        out = fn()
        e1.record(self.stream)
        torch.cuda.synchronize()
        self.barrier()
        return self.max_over_ranks(e0.elapsed_time(e1)), out

    def run_steps(self, items, fn, concurrency):
        """fn(item) for every item, `concurrency` in flight (one stream and
        native context per worker); returns the summed kernel launches."""
        from paper_1908_02461_b200 import _native
        from paper_1908_02461_b200 import batch as PB
        local = self.local

        def one(i):
            fn(items[i])
            return _native.context(local).last_launches
        return sum(PB._run(one, len(items), concurrency, self.dev))

    # ------------------------------------------------------------ headline c3
    def c3(self):
        import paper_1908_02461_b200 as P
        from paper_1908_02461_b200 import _native
        from paper_1908_02461_b200 import batch as PB
        torch, args = self.torch, self.args
        conc = max(1, args.concurrency)
        imgs = [workload(args, self.rank, j) for j in range(conc)]
        xs_dev = [torch.from_numpy(im.x).to(self.dev) for im in imgs]
        x_dev = xs_dev[0]
        cfg = P.TunerConfig()
        ctx = _native.context(self.local)

        def step(x):
            return P.atsfft2d_arrays(x, cfg, args.est_loops, 11, precision=args.precision)

        for _ in range(max(args.warmup, 1)):
            (ij, vals), state = step(x_dev)
        for j in range(conc):
            PB.warm_workers(lambda j=j: step(xs_dev[j]), conc, self.dev)
        self.run_steps([xs_dev[i % conc] for i in range(max(args.warmup, 2 * conc))], step, conc)
        torch.cuda.synchronize()
        parity = None
        g = golden("c3_ats")
        if self.rank == 0 and args.n == 4096 and args.k == 100 and args.snr == 20.0 and g:
            parity = compare(ij.cpu().numpy() if hasattr(ij, "cpu") else ij,
                             vals.cpu().numpy() if hasattr(vals, "cpu") else vals, g,
                             args.precision, state)

        gc.disable()
        sampler = ClockSampler(self.nvml_index)
        sampler.start()
        ms_max, launches = self.timed(lambda: self.run_steps(
            [xs_dev[i % conc] for i in range(args.steps)], step, conc))
        clocks = sampler.stop()
        value = self.world * args.steps / (ms_max / 1e3)
        lat_ms, _ = self.timed(lambda: self.run_steps([x_dev] * args.steps, step, 1))
        latency = {"ms_per_transform": lat_ms / args.steps,
                   "transforms_per_s": self.world * args.steps / (lat_ms / 1e3), "in_flight": 1}

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

            self.run_steps(hosts, step_host, conc)
            d2h[0] = 0
            e2e_ms, _ = self.timed(lambda: self.run_steps(
                [hosts[i % conc] for i in range(args.steps)], step_host, conc))
            nperm = cfg.iters(args.n) + 2 + args.est_loops
            e2e = {"value": self.world * args.steps / (e2e_ms / 1e3), "unit": UNIT, "in_flight": conc,
                   "h2d_bytes_per_step": args.n * args.n * 8 + nperm * 48,
                   "d2h_bytes_per_step": d2h[0] // max(args.steps, 1)}
        gc.enable()

        roofline, kernels = self.roofline(step, x_dev, f"c3/{args.precision}", value,
                                          latency["ms_per_transform"])

        # dense cuFFT of the same image, for context only
        xc = x_dev.to(torch.complex64)
        for _ in range(3):
            torch.fft.fft2(xc)
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(self.stream)
        for _ in range(10):
            torch.fft.fft2(xc)
        c1.record(self.stream)
        torch.cuda.synchronize()
        self.c3_img = imgs[0]
        del xs_dev, x_dev, xc
        return dict(value=value, ms_max=ms_max, launches=launches, clocks=clocks, latency=latency,
                    e2e=e2e, roofline=roofline, kernels=kernels, parity=parity,
                    cufft_ms=c0.elapsed_time(c1) / 10, state=state, conc=conc)

    def roofline(self, step, x, traffic_key, value, single_ms):
        """Kernel-level + transform-level roofline from an instrumented pass of
        the same workload (library per-launch CUDA events on the launching
        stream, algorithmic bytes per DESIGN.md §3)."""
        from paper_1908_02461_b200 import _native
        torch, args = self.torch, self.args
        ctx = _native.context(self.local)
        # one instrumented pass first (event pool, serialised-stream path warm),
        # discarded; the report below covers the nprof passes after it
        ctx.set_profiling(True)
        step(x)
        torch.cuda.synchronize()
        ctx.set_profiling(False)
        ctx.set_profiling(True)
        nprof = max(1, min(args.profile_steps, args.steps))
        pe0 = torch.cuda.Event(enable_timing=True)
        pe1 = torch.cuda.Event(enable_timing=True)
        pe0.record(self.stream)
        for _ in range(nprof):
            step(x)
        pe1.record(self.stream)
        torch.cuda.synchronize()
        rep = ctx.profile_report()
        ctx.set_profiling(False)
        prof_ms = pe0.elapsed_time(pe1)
        peak, peak_kind = peaks()
        if not rep:
            return None, {}
        # dominant kernel of the HBM roofline: the one moving the most
        # algorithmic bytes per step (the per-launch event brackets add a few
        # microseconds to every launch, which would rank the latency-bound
        # small kernels first by time; the longest kernel is reported beside it)
        name, (cnt, tms, tbytes) = max(rep.items(), key=lambda kv: kv[1][2])
        tname, (tcnt, ttms, ttbytes) = max(rep.items(), key=lambda kv: kv[1][1])
        achieved = (tbytes / cnt) / (tms / cnt / 1e3) / 1e9
        traffic = kernel_traffic(traffic_key).get(name)
        bytes_tr = sum(v[2] for v in rep.values()) / nprof
        roof = {
            "bound": "hbm", "kernel": name, "selection": "most algorithmic bytes per step",
            "longest_kernel": {"kernel": tname, "share_of_step": ttms / prof_ms,
                               "avg_launch_us": ttms / tcnt * 1e3,
                               "achieved_GBps": (ttbytes / tcnt) / (ttms / tcnt / 1e3) / 1e9},
            "achieved": achieved, "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "traffic_source": (f"profiles/kernel_traffic.json {traffic_key} (ncu --set full)"
                               if traffic is not None else None),
            "alg_bytes_per_launch": tbytes / cnt, "launches_per_step": cnt / nprof,
            "avg_launch_us": tms / cnt * 1e3, "share_of_step": tms / prof_ms,
            "transform": {
                "alg_bytes_per_transform": bytes_tr,
                "achieved_in_flight": bytes_tr * value / self.world / 1e9,
                "frac_in_flight": bytes_tr * value / self.world / 1e9 / peak,
                "achieved_single": bytes_tr / (single_ms / 1e3) / 1e9,
                "frac_single": bytes_tr / (single_ms / 1e3) / 1e9 / peak,
                "note": "sum of every kernel's algorithmic bytes (DESIGN.md §3) per transform"},
        }
        kernels = {k: {"launches_per_step": v[0] / nprof, "ms_per_step": v[1] / nprof,
                       "GBps": (v[2] / v[1] / 1e6) if v[1] > 0 else None}
                   for k, v in sorted(rep.items(), key=lambda kv: -kv[1][1])[:10]}
        return roof, kernels

    # ------------------------------------------------------------ other legs
    def leg_c3_fp64(self):
        """c3 in the fp64 verification precision (the reference's arithmetic)."""
        import paper_1908_02461_b200 as P
        torch, args = self.torch, self.args
        conc = max(1, args.concurrency)
        steps = max(1, min(args.steps, 60))
        xs = [torch.from_numpy(workload(args, self.rank, j).x).to(self.dev) for j in range(conc)]
        cfg = P.TunerConfig()

        def step(x):
            return P.atsfft2d_arrays(x, cfg, args.est_loops, 11, precision="fp64")

        (ij, vals), state = step(xs[0])
        # every worker's native context allocates its fp64 workspace before the
        # timed region (a pool thread that got no warm-up item would grow it there)
        from paper_1908_02461_b200 import batch as PB
        PB.warm_workers(lambda: step(xs[0]), conc, self.dev)
        self.run_steps([xs[i % conc] for i in range(2 * conc)], step, conc)
        g = golden("c3_ats")
        parity = compare(ij, vals, g, "fp64", state) if (self.rank == 0 and g and args.n == 4096
                                                          and args.k == 100 and args.snr == 20.0) else None
        ms, _ = self.timed(lambda: self.run_steps([xs[i % conc] for i in range(steps)], step, conc))
        lat, _ = self.timed(lambda: self.run_steps([xs[0]] * steps, step, 1))
        value = self.world * steps / (ms / 1e3)
        roof, kernels = self.roofline(step, xs[0], "c3/fp64", value, lat / steps)
        return {"workload": "c3 in fp64 (verification mode, the reference's float64 arithmetic)",
                "value": value, "unit": UNIT, "in_flight": conc,
                "steps": steps, "ms_per_transform_single": lat / steps, "parity": parity,
                "roofline": roof, "kernels": kernels, "scaling": "weak"}

    def _small_leg(self, x, fn, steps, gold, precision, conc, ats):
        torch = self.torch
        out = fn(x)
        for _ in range(3):
            fn(x)
        from paper_1908_02461_b200 import batch as PB
        PB.warm_workers(lambda: fn(x), conc, self.dev)   # every worker context warm
        self.run_steps([x] * (2 * conc), fn, conc)
        parity = None
        if self.rank == 0 and gold is not None:
            (ij, vals), state = out if ats else (out, None)
            parity = compare(ij, vals, gold, precision, state)
        torch.cuda.synchronize()
        ms, _ = self.timed(lambda: self.run_steps([x] * steps, fn, conc))
        lat, _ = self.timed(lambda: self.run_steps([x] * steps, fn, 1))
        return {"value": self.world * steps / (ms / 1e3), "unit": UNIT, "in_flight": conc,
                "steps": steps, "ms_per_transform_single": lat / steps, "parity": parity,
                "scaling": "weak", "parallelism": f"independent transforms, {self.world} rank(s)"}

    def leg_c1(self):
        """configs[0]: SFFT with known k, 256^2 complex128, k=10, noiseless
        (the reference's generate_planted image, stored in the c1 golden)."""
        import paper_1908_02461_b200 as P
        g = golden("c1_sfft")
        if g is None:
            return {"skipped": "tests/golden/c1_sfft.npz missing"}
        cfg = P.SfftConfig(n=256, k=10)
        x = self.torch.from_numpy(g["x"]).to(self.dev)
        steps = max(1, min(self.args.steps, 200))
        out = {"workload": "c1: SFFT known k, 256x256 complex128, k=10, noiseless, L=8, B=64 (fp64)"}
        out.update(self._small_leg(x, lambda xx: P.sfft2d_arrays(xx, cfg, int(g["cfg"][5]),
                                                                 precision="fp64"),
                                   steps, g, "fp64", self.args.concurrency, ats=False))
        return out

    def leg_c2(self):
        """configs[1]: ATSFFT 1024^2 complex64, k=50, 30 dB (fp32)."""
        import paper_1908_02461_b200 as P
        g = golden("c2_ats")
        from paper_1908_02461_b200.signals import sparse_image
        x = self.torch.from_numpy(sparse_image(1024, 50, 7, snr_db=30.0).x).to(self.dev)
        cfg = P.TunerConfig()
        steps = max(1, min(self.args.steps, 200))
        out = {"workload": "c2: ATSFFT 1024x1024 complex64, k=50, 30 dB, est_loops=8 (fp32)"}
        out.update(self._small_leg(x, lambda xx: P.atsfft2d_arrays(xx, cfg, 8, 11, precision="fp32"),
                                   steps, g, "fp32", self.args.concurrency, ats=True))
        return out

    def leg_c4(self):
        """configs[3]: 2048 independent 1024^2 c64 images, per-image seed,
        k ~ U[20, 200], log-uniform magnitudes, 25 dB, sharded over the ranks
        (contiguous shards, no data-path collective; strong scaling).  Images
        0..11 are the host-generated images pinned by the reference goldens
        (tests/golden/c4b_*.npz, parity-checked from this timed batch); the
        rest are built in HBM by the device generator."""
        import paper_1908_02461_b200 as P
        from paper_1908_02461_b200 import distributed as D
        from paper_1908_02461_b200.signals import device_sparse_image, sparse_image
        torch, args = self.torch, self.args
        total = args.c4_images
        idx = D.batch_shard(total, self.rank, self.world)
        xs, seeds, pinned = [], [], []
        t0 = time.perf_counter()
        for i in idx:
            seed, k = c4_params(i)
            g = golden(f"c4b_{i:02d}") if i < 12 else None
            if g is not None:
                im = sparse_image(1024, k, seed, snr_db=25.0, magnitude="loguniform")
                xs.append(torch.from_numpy(im.x).to(self.dev))
                pinned.append((len(xs) - 1, g))
            else:
                xs.append(device_sparse_image(1024, k, seed, snr_db=25.0, magnitude="loguniform",
                                              device=self.dev).x)
            seeds.append(1 + i)
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - t0
        cfg = P.TunerConfig()
        conc = args.concurrency

        def run():
            return P.atsfft2d_batch(xs, cfg, 8, seeds, concurrency=conc, precision="fp32", arrays=True)

        run()
        samples, res = [], None
        sampler = ClockSampler(self.nvml_index)
        sampler.start()
        for _ in range(2):
            ms, res = self.timed(run)
            samples.append(total / (ms / 1e3))
        clocks = sampler.stop()
        parity = None
        if pinned:
            checks = [compare(res[j][0][0], res[j][0][1], g, "fp32", res[j][1]) for j, g in pinned]
            parity = {"images_checked": len(checks),
                      "all_within_tolerance": all(c["within_tolerance"] for c in checks),
                      "support_equal": sum(c["support_equal"] for c in checks),
                      "max_rel_err": max(c["max_rel_err"] for c in checks)}
        return {"workload": f"c4: {total} independent 1024x1024 c64 images, k~U[20,200], log-uniform "
                            "magnitudes, 25 dB, est_loops=8, fp32; images 0-11 host-generated and "
                            "pinned to the reference, the rest from the device generator",
                "value": float(np.median(samples)), "samples": samples, "unit": UNIT,
                "scaling": "strong", "concurrency": conc, "images_per_rank": len(idx),
                "parallelism": f"batch sharded over {self.world} rank(s), no data-path collective",
                "generation_s": gen_s, "clocks": clocks, "parity": parity}

    def leg_c5(self):
        """configs[4]: 16384^2 c64 (2 GiB), 20% of the k coefficients in the
        64x64 wrap-around DC block, unit magnitude, 15 dB, ATSFFT.  The tuner
        passes are sequential and the estimation now reads the dense spectrum
        (k_estimate_conv at b_estimate = 8192, x_hat itself at N): nothing of
        one transform is left to split, so at N > 1 every rank runs its own
        transform (replicas, weak scaling).  Images from the
        device generator (the reference-pinned c5 cases are GPU tests)."""
        import paper_1908_02461_b200 as P
        from paper_1908_02461_b200.signals import device_sparse_image
        torch = self.torch
        ks = [int(v) for v in self.args.c5_ks.split(",") if v.strip()]
        cfg = P.TunerConfig()
        buf = torch.empty((16384, 16384), dtype=torch.complex64, device=self.dev)
        out = {"workload": "c5: ATSFFT 16384x16384 complex64, 20% of k in the 64x64 DC block, 15 dB, "
                           "est_loops=8, fp32, device-generated",
               "parallelism": f"replicas: one transform per rank, {self.world} rank(s)",
               "scaling": "weak", "per_k": {}}
        for k in ks:
            img = device_sparse_image(16384, k, 5 + 1000 * self.rank, snr_db=15.0, cluster_frac=0.2,
                                      cluster_side=64, device=self.dev, out=buf)

            def one():   # device-resident arrays, like the c3 value leg
                return P.atsfft2d_arrays(img.x, cfg, 8, 6, precision="fp32")
            (ij, vals), state = one()
            one()
            reps = 3
            ms, _ = self.timed(lambda: [one() for _ in range(reps)])
            res = {tuple(key): True for key in np.asarray(ij).tolist()}
            truth = img.truth
            out["per_k"][str(k)] = {
                "ms_per_transform": ms / reps, "transforms_per_s": self.world * reps / (ms / 1e3),
                "detected_k": state.detected_k, "b_estimate": state.b_estimate,
                "passes": len(state.history), "recovered": len(res),
                "planted_recovered": sum(1 for key in truth if key in res) / max(len(truth), 1)}
        out["parity"] = ("device-generated images are timed here; the host-generated c5 images "
                         "(k = 64, 256, 1024, 4096) are pinned to the reference goldens by "
                         "tests/test_gpu_parity.py::test_c5_atsfft_vs_reference / test_c5_sweep_vs_reference")
        del buf
        return out

    def leg_c3_sfft(self):
        """Known-k SFFT on the c3 image (B = 128, L = 8): location loops and
        estimation loops split over the ranks (sfft2d_loopsplit: vote-count
        all-reduce + estimate all-reduce), parity vs the reference golden."""
        import paper_1908_02461_b200 as P
        from paper_1908_02461_b200 import distributed as D
        from paper_1908_02461_b200.signals import sparse_image
        torch = self.torch
        g = golden("c3_sfft")
        x = torch.from_numpy(sparse_image(4096, 100, 7, snr_db=20.0).x).to(self.dev)
        cfg = P.SfftConfig(n=4096, k=100)
        seed = int(g["cfg"][5]) if g is not None else 12

        def one():
            if self.world > 1:
                return D.sfft2d_loopsplit(x, cfg, seed, precision="fp32")
            return P.sfft2d(x, cfg, seed, precision="fp32")
        res = one()
        for _ in range(3):
            one()
        reps = max(3, min(self.args.steps, 50))
        ms, _ = self.timed(lambda: [one() for _ in range(reps)])
        parity = None
        if self.rank == 0 and g is not None:
            keys = list(res)
            parity = compare(np.array(keys).reshape(-1, 2), np.array([res[k] for k in keys]), g, "fp32")
        return {"workload": "c3 image, SFFT with known k=100 (B=128, L=8), fp32",
                "ms_per_transform": ms / reps, "transforms_per_s": reps / (ms / 1e3),
                "parallelism": (f"location + estimation loops split over {self.world} rank(s)"
                                if self.world > 1 else "1 rank"), "scaling": "strong",
                "parity": parity}


def c3_config(args) -> dict:
    """The workload both arms report (BASELINE.json configs[2])."""
    return {"workload": f"c3: ATSFFT {args.n}x{args.n} complex64, k={args.k}, {args.snr:g} dB SNR, "
                        f"TunerConfig() defaults, est_loops={args.est_loops}, one transform per step",
            "l2": "inputs larger than L2 (134 MB image)"}


def cpu_baseline(x, args):
    from oracle import sfft_oracle as O
    O.FAST = True
    t0 = time.perf_counter()
    O.atsfft(x, O.TunerParams(), args.est_loops, 11)
    dt = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"one full ATSFFT transform of the c3 image ({args.n}^2 c64, k={args.k}, "
                      f"{args.snr:g} dB, est_loops={args.est_loops}) by the numpy oracle port "
                      f"(pocketfft FFTs), 1 thread, {dt:.1f} s"}


def main_ours(args):
    b = Bench(args)
    c3 = b.c3()
    legs = {}
    want = [] if args.legs == "none" else [v.strip() for v in args.legs.split(",") if v.strip()]
    for name in want:
        fn = getattr(b, f"leg_{name}", None)
        if fn is None:
            legs[name] = {"skipped": "unknown leg"}
            continue
        t0 = time.perf_counter()
        try:
            legs[name] = fn()
        except Exception as e:  # noqa: BLE001 - a failing leg is reported, not hidden
            legs[name] = {"error": f"{type(e).__name__}: {e}"}
        legs[name]["wall_s"] = time.perf_counter() - t0
        b.torch.cuda.synchronize()
        b.torch.cuda.empty_cache()
    cpu = None
    if b.rank == 0 and b.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(b.c3_img.x, args)
    if b.rank == 0:
        st = c3["state"]
        line = {
            "metric": METRIC, "value": c3["value"], "unit": UNIT, "n_gpus": b.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": c3["ms_max"] / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == "fp32" else "f64", "data": "synthetic",
            "config": c3_config(args),
            "execution": {"precision": args.precision,
                          "in_flight": f"{c3['conc']} distinct images, {c3['conc']} transforms in "
                                       "flight (one CUDA stream + native context each)",
                          "parallelism": (f"replicas: independent c3 transforms on each of {b.world} "
                                          "rank(s) (the ATSFFT tuner passes are sequential and c3's "
                                          "b_estimate = N leaves nothing to split; DESIGN.md §6)")},
            "e2e": c3["e2e"], "latency": c3["latency"], "roofline": c3["roofline"],
            "cpu_baseline": cpu, "clocks": c3["clocks"], "gpu_launches": c3["launches"],
            "kernels": c3["kernels"], "parity": c3["parity"], "legs": legs,
            "context": {"cufft_dense_fft2_c64_ms": c3["cufft_ms"], "detected_k": st.detected_k,
                        "passes": st.passes, "trajectory": [bb for bb, _, _ in st.history]},
        }
        print(json.dumps(line), flush=True)
    if b.world > 1:
        b.dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------- reference arm
def _port_worker(args_tuple):
    from oracle import sfft_oracle as O
    O.FAST = True
    x, est_loops, seed = args_tuple
    t0 = time.perf_counter()
    O.atsfft(x, O.TunerParams(), est_loops, seed)
    return time.perf_counter() - t0


def _refpkg_worker(job):
    """One timed call of the UNMODIFIED reference package (baseline/_ref)."""
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    import sfft2d as ref
    name, reps = job
    if name == "c1":
        sig = ref.generate_planted(256, 10, 1)
        x, call = sig.x, (lambda: ref.sfft2d(sig.x, ref.SfftConfig(n=256, k=10), 2))
    else:
        from paper_1908_02461_b200.signals import sparse_image
        if name == "c2":
            x = sparse_image(1024, 50, 7, snr_db=30.0).x
        else:
            x = sparse_image(4096, 100, 7, snr_db=20.0).x
        call = (lambda: ref.atsfft2d(x, ref.TunerConfig(), 8, 11))
    # windows pre-warmed as the reference's own harness does (bench.py:110-116)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    return name, times


def run_reference(args):
    """The reference arm: K steps, a step = one full c3 transform by the
    numpy oracle port, spread over the host's cores (one process each), plus
    the UNMODIFIED reference package (baseline/_ref) on c1, c2 and c3 in the
    same pool.  Same metric, unit and config as our arm."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import multiprocessing as mp
    img = workload(args, 0)
    cores = os.cpu_count() or 1
    procs = max(1, min(cores, 16, args.steps))
    steps = args.steps
    ctx = mp.get_context("fork")
    refpkg = None
    have_pkg = os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "sfft2d"))
    t_all = time.perf_counter()
    with ctx.Pool(procs) as pool:
        pend = None
        if have_pkg:
            # the unmodified reference, one process per config, alongside the
            # port's steps (c3 alone is ~2 min on one core, so it runs once)
            pend = pool.map_async(_refpkg_worker, [("c3", 1), ("c1", 3), ("c2", 3)], chunksize=1)
        # warm-up: one untimed transform per worker process (W > 0)
        if args.warmup > 0:
            pool.map(_port_worker, [(img.x, args.est_loops, 11)] * procs, chunksize=1)
        t0 = time.perf_counter()
        times = pool.map(_port_worker, [(img.x, args.est_loops, 11)] * steps, chunksize=1)
        dt = time.perf_counter() - t0
        if pend is not None:
            got = dict(pend.get())
            refpkg = {"source": "baseline/_ref (pip --no-deps install of /root/reference/pkg, "
                                "unmodified), 1 process per config, 1 thread each",
                      "per_config": {k: {"seconds_per_transform": float(np.median(v)),
                                         "transforms_per_s": 1.0 / float(np.median(v)),
                                         "reps": len(v)} for k, v in got.items()}}
    value = steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": args.warmup,
        "ms_per_step": dt / steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": c3_config(args),
        "execution": f"{steps} transforms over {procs} host processes (1 thread each)",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "port",
                         "cpu_model": cpu_model(), "host_cpus": cores,
                         "seconds_per_transform_median": float(np.median(times)),
                         "sample": f"{steps} full c3 transforms of the numpy oracle port "
                                   f"(pocketfft FFTs) on {procs} processes"},
        "reference_package": refpkg,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.impl == "reference":
        return run_reference(args)
    return main_ours(args)


if __name__ == "__main__":
    sys.exit(main())
