"""Algorithm 2 (ATSFFT: sparsity detection by adaptive bin tuning) — mirror of
``/root/reference/pkg/src/sfft2d/tuner.py`` on the sm_100a path.

The tuning loop itself runs natively (csrc/capi.cu ``run_ats``): each pass is a
fold + bucket FFT (or, at B = N, a permuted view of one dense |x_hat|), a
local-maximum count with ordered compaction, and the vote-histogram update;
the host controller applies the ratio rule / cycle guard / confirmation
passes of tuner.py:182-226 between passes (one host sync per pass).

Permutations come from the caller's Generator in the reference order: the
native controller draws them on demand through the Generator's bitgen_t with
numpy's own bounded-integer routine, so the caller's Generator advances
exactly as under the reference.
"""

from __future__ import annotations

import ctypes
import math
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._tensors import as_device_image
from .engine import ConfigurationError, SfftConfig, _fetch, _nearest_pow2, _stream, default_bins, to_dict
from .hashing import WindowCache, draw_permutation, is_power_of_two

__all__ = ["TunerConfig", "TunerState", "count_local_maxima", "update_bins", "detect_sparsity",
           "atsfft2d", "atsfft2d_arrays"]


@dataclass
class TunerConfig:
    """Adaptive tuning parameters (tuner.py:47-78)."""

    b0: int = 16
    eps1: float = 0.5
    eps2: float = 1.0
    delta1: float = 0.02
    delta2: float = 0.05
    max_tuning_iters: int | None = None
    mag_floor: float = 1e-3
    window_delta_pass: float = 1e-3
    window_delta_stop: float = 1e-8
    gain_floor: float = 1e-6
    prune_rel: float = 1e-3

    def __post_init__(self):
        if not (0.0 < self.delta1 < self.delta2 < 1.0):
            raise ConfigurationError("need 0 < delta1 < delta2 < 1")
        if not (0.0 < self.eps1 < 1.0) or self.eps2 <= 0.0:
            raise ConfigurationError("need 0 < eps1 < 1 and eps2 > 0")
        if not is_power_of_two(self.b0):
            raise ConfigurationError(f"b0 {self.b0} is not a power of 2")

    def iters(self, n: int) -> int:
        if self.max_tuning_iters is not None:
            return self.max_tuning_iters
        return 2 * max(int(math.log2(n)), 1)

    def _c(self) -> _native.TunerCfg:
        return _native.TunerCfg(
            self.b0, -1 if self.max_tuning_iters is None else int(self.max_tuning_iters),
            self.eps1, self.eps2, self.delta1, self.delta2, self.mag_floor,
            self.window_delta_pass, self.window_delta_stop, self.gain_floor, self.prune_rel)


@dataclass
class TunerState:
    """Trajectory of the adaptive iteration (tuner.py:81-94)."""

    history: list = field(default_factory=list)  # (bins, count, ratio or None)
    converged: bool = False
    detected_k: int = 0
    b_detect: int = 0
    b_estimate: int = 0
    vote_passes: int = 0

    @property
    def passes(self) -> int:
        return len(self.history)


def _state(sc: _native.TunerStateC) -> TunerState:
    n = sc.passes
    # one slice per ctypes array (element-wise indexing costs ~0.1 us per access)
    hist = [(int(b), int(c), float(r) if h else None)
            for b, c, r, h in zip(sc.hist_bins[:n], sc.hist_count[:n], sc.hist_ratio[:n],
                                  sc.hist_has_ratio[:n])]
    st = TunerState(history=hist, converged=bool(sc.converged), detected_k=int(sc.detected_k),
                    b_detect=int(sc.b_detect), b_estimate=int(sc.b_estimate),
                    vote_passes=int(sc.vote_passes))
    st.pass_us = sc.hist_us[:n]   # diagnostic, not compared
    st.n_candidates = int(sc.n_candidates)   # diagnostic: coordinates estimated
    return st


_seeded = threading.local()


def _generator(rng):
    """``np.random.default_rng(rng)`` for the native draws.  An int seed reuses
    this thread's Generator for that seed, reset to the seed's initial state
    (1.5 us instead of 15.5 us for SeedSequence hashing); the draws are the
    same stream.  Returns (generator, bitgen pointer, snapshot-or-None)."""
    if isinstance(rng, np.random.Generator):
        return rng, rng.bit_generator.ctypes.bit_generator.value, rng.bit_generator.state
    if isinstance(rng, (int, np.integer)) and not isinstance(rng, bool) and rng >= 0:
        cache = getattr(_seeded, "gens", None)
        if cache is None:
            cache = _seeded.gens = {}
        hit = cache.get(int(rng))
        if hit is None:
            gen = np.random.default_rng(int(rng))
            hit = cache[int(rng)] = (gen, gen.bit_generator.state,
                                     gen.bit_generator.ctypes.bit_generator.value)
            if len(cache) > 256:
                cache.pop(next(iter(cache)))
        else:
            hit[0].bit_generator.state = hit[1]
        return hit[0], hit[2], None
    gen = np.random.default_rng(rng)
    return gen, gen.bit_generator.ctypes.bit_generator.value, None


def update_bins(b: int, r: float, cfg: TunerConfig, n: int) -> int:
    """Shrink below delta1, hold inside the band, grow at or above delta2,
    snapped to a power of two in [4, n] (tuner.py:121-130)."""
    if r < cfg.delta1:
        scaled = b * cfg.eps1
    elif r < cfg.delta2:
        scaled = float(b)
    else:
        scaled = b * (1.0 + cfg.eps2)
    return max(4, min(_nearest_pow2(scaled), n))


def count_local_maxima(bins, mag_floor: float, *, precision: str = "fp64", device=None):
    """Bins strictly above all 8 toroidal neighbours and above
    ``mag_floor * max|Z|`` (tuner.py:97-118), computed on the GPU.  Returns the
    count and an (m, 2) int64 array of bin coordinates in row-major order."""
    torch = _native._torch()
    if _is_tensor(bins):
        t = bins
        if t.dim() != 2 or t.shape[0] != t.shape[1]:
            raise ValueError(f"expected a square bin grid, got {tuple(t.shape)}")
    else:
        a = np.asarray(bins)
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError(f"expected a square bin grid, got {a.shape}")
        t = None
    b = int((t if t is not None else a).shape[0])
    if b < 4:
        raise ValueError("bin grid must be at least 4x4")
    prec = _native.precision_code(precision)
    cdt = torch.complex128 if prec == _native.FP64 else torch.complex64
    if t is None:
        dev = torch.cuda.current_device() if device is None else int(device)
        t = torch.from_numpy(np.ascontiguousarray(a.astype(np.complex128))).to(f"cuda:{dev}")
    t = t.to(cdt).contiguous()
    ctx = _native.context(t.device.index)
    out = torch.empty(b * b // 4 + 64, dtype=torch.int32, device=t.device)
    cnt = ctypes.c_int64()
    with torch.cuda.device(t.device.index):
        st = _stream(torch, t.device.index)
        ctx.check(ctx.lib.sfft2d_local_maxima(ctx.handle, t.data_ptr(), b, float(mag_floor), prec,
                                              ctypes.byref(cnt), out.data_ptr(), out.numel(), st))
        torch.cuda.current_stream(t.device.index).synchronize()
    flat = out[: cnt.value].cpu().numpy().astype(np.int64)
    return int(cnt.value), np.stack([flat // b, flat % b], axis=1)


def _is_tensor(x) -> bool:
    from ._tensors import is_torch_tensor
    return is_torch_tensor(x)


def reconcile_generator(gen, snapshot, n: int, drawn: int, used: int) -> None:
    """The speculative fold draws the next pass's permutation before the tuner
    knows whether a next pass or an estimation loop will consume it; when none
    did (drawn > used), put the caller's Generator where the reference leaves
    it: back to the call's snapshot, then replay the `used` permutation draws
    (hashing.draw_permutation = the reference's four integers() calls)."""
    if drawn <= used:
        return
    gen.bit_generator.state = snapshot
    for _ in range(used):
        draw_permutation(n, gen)


def _run_ats(x, cfg: TunerConfig, est_loops: int, rng, precision, device, estimate: bool,
             on_device: bool = False):
    torch = _native._torch()
    img = as_device_image(x, device, upload=on_device)
    n = img.n
    prec = _native.precision_code(precision)
    # The native controller draws each permutation on demand from this
    # Generator's own bit generator with numpy's bounded-integer routine, so a
    # caller's Generator advances exactly as under the reference.
    gen, bitgen, snapshot = _generator(rng)
    ctx = _native.context(img.device)
    ctx.ensure_tables(n, cfg.window_delta_pass, cfg.window_delta_stop)
    ccfg = cfg._c()
    sc = _native.TunerStateC()
    res = _native.ResultC()
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)
        if img.tensor is not None:
            ptr, on_host = img.tensor.data_ptr(), 0
        else:
            ptr, on_host = img.host.ctypes.data, 1
        t_call = time.perf_counter()
        if estimate:
            rc = ctx.lib.sfft2d_atsfft_bitgen(ctx.handle, ptr, img.dtype_code, on_host, n,
                                              ctypes.byref(ccfg), int(est_loops), bitgen, prec, st,
                                              ctypes.byref(res), ctypes.byref(sc))
        else:
            rc = ctx.lib.sfft2d_detect_sparsity_bitgen(ctx.handle, ptr, img.dtype_code, on_host, n,
                                                       ctypes.byref(ccfg), bitgen, prec, st,
                                                       ctypes.byref(sc))
        ctx.last_call_us = (time.perf_counter() - t_call) * 1e6
        if rc == _native.ERR_VALUE and snapshot is not None:
            gen.bit_generator.state = snapshot   # the reference validates x before drawing
        elif rc in (_native.OK, _native.ERR_CONFIG) and snapshot is not None:
            reconcile_generator(gen, snapshot, n, int(sc.perms_drawn), int(sc.perms_used))
        ctx.check(rc)
        ctx.last_launches = int(res.gpu_launches)
        state = _state(sc)
        if not estimate:
            nv = int(sc.n_votes)
            if on_device:   # keys / tallies stay in device tensors (distributed split)
                kd = torch.empty(max(nv, 1), dtype=torch.int32, device=img.tensor.device)
                td = torch.empty(max(nv, 1), dtype=torch.int32, device=img.tensor.device)
                if nv:
                    ctx.check(ctx.lib.sfft2d_fetch_votes(ctx.handle, kd.data_ptr(), td.data_ptr(),
                                                         0, st))
                return state, (kd[:nv], td[:nv])
            keys = np.empty(nv, dtype=np.int32)
            tallies = np.empty(nv, dtype=np.int32)
            if nv:
                ctx.check(ctx.lib.sfft2d_fetch_votes(ctx.handle, keys.ctypes.data,
                                                     tallies.ctypes.data, 1, st))
            k64 = keys.astype(np.int64)
            coords = np.stack([k64 // n, k64 % n], axis=1) if nv else np.empty((0, 2), np.int64)
            return state, (coords, tallies.astype(np.int64))
        ij, vals = _fetch(ctx, res, st, prec)
    return (ij, vals), state


def detect_sparsity(x, cfg: TunerConfig, rng, *, cache: WindowCache | None = None,
                    precision: str = "fp64", device=None):
    """Adaptive tuning loop with vote accumulation (tuner.py:142-241).
    Returns (TunerState, (coords int64[m, 2], tallies int64[m]))."""
    return _run_ats(x, cfg, 0, rng, precision, device, estimate=False)


def atsfft2d_arrays(x, cfg: TunerConfig, est_loops: int, rng, *,
                    cache: WindowCache | None = None, precision: str = "fp64", device=None):
    """``atsfft2d`` returning ((coords, values), state) instead of a dict."""
    return _run_ats(x, cfg, est_loops, rng, precision, device, estimate=True)


def atsfft2d(x, cfg: TunerConfig, est_loops: int, rng, *, cache: WindowCache | None = None,
             precision: str = "fp64", device=None):
    """Sparse transform without prior sparsity: detect, vote, estimate
    (tuner.py:244-282).  Returns (dict, TunerState)."""
    (ij, vals), state = atsfft2d_arrays(x, cfg, est_loops, rng, cache=cache, precision=precision,
                                        device=device)
    return to_dict(ij, vals), state


# re-exported for API parity with the reference module
__all__ += ["SfftConfig", "default_bins"]
