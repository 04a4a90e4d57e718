"""Algorithm 1 (fixed-sparsity 2D SFFT) — mirror of
``/root/reference/pkg/src/sfft2d/engine.py`` on the sm_100a path.

``sfft2d`` keeps the reference signature and result (a dict ``(i, j) ->
complex``).  The host draws the 2L per-loop permutation streams exactly as the
reference does (engine.py:266-268, 280) and hands them to the native
controller ``sfft2d_sfft`` (csrc/capi.cu ``run_sfft``): one fused fold of all L
location loops, bucket FFTs, top-2k selection, unhash + dedup vote histogram,
threshold compaction, L estimation loops, median, top-k, prune.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from ._tensors import as_device_image
from .hashing import (FlatWindow, WindowCache, build_flat_window, draw_permutation,
                      is_power_of_two)

__all__ = ["ConfigurationError", "SfftConfig", "default_bins", "sfft2d", "sfft2d_arrays"]


class ConfigurationError(ValueError):
    """Raised when a transform configuration cannot be executed (engine.py:45-46)."""


def _nearest_pow2(v: float) -> int:
    """Power of two nearest to v, ties to the lower one (engine.py:49-52)."""
    lo = 1 << max(int(math.floor(math.log2(v))), 0) if v >= 1 else 1
    return lo if (v - lo) <= (2 * lo - v) else 2 * lo


def default_bins(n: int, k: int) -> int:
    """Nearest power of two to sqrt(min(n, 256) * k), clamped to [4, n] (engine.py:55-66)."""
    k = max(k, 1)
    return max(4, min(_nearest_pow2(math.sqrt(min(n, 256) * k)), n))


_WINDOWS = WindowCache()


@dataclass
class SfftConfig:
    """Inputs of the fixed-sparsity transform (engine.py:69-119)."""

    n: int
    k: int
    loops: int = 8
    d_factor: int = 2
    vote_threshold: int | None = None
    b_bins: int | None = None
    window_delta_pass: float = 1e-3
    window_delta_stop: float = 1e-8
    gain_floor: float = 1e-6
    prune_rel: float = 1e-3

    def __post_init__(self):
        if not is_power_of_two(self.n):
            raise ConfigurationError(f"side {self.n} is not a power of 2")
        if self.k < 0 or self.k > self.n * self.n:
            raise ConfigurationError(f"sparsity {self.k} out of range for n={self.n}")
        if self.loops < 1:
            raise ConfigurationError("loops must be >= 1")
        if self.b_bins is None:
            self.b_bins = default_bins(self.n, self.k)
        b = self.b_bins
        if not is_power_of_two(b) or b > self.n or self.n % b != 0:
            raise ConfigurationError(f"bin count {b} must be a power of 2 dividing {self.n}")
        if self.vote_threshold is None:
            self.vote_threshold = (self.loops + 1) // 2
        if not 1 <= self.vote_threshold <= self.loops:
            raise ConfigurationError(
                f"vote_threshold {self.vote_threshold} outside [1, {self.loops}]")
        if self.num_kept_bins > b * b:
            raise ConfigurationError(
                f"d_factor*k = {self.num_kept_bins} exceeds the {b}x{b} bin budget")

    @property
    def num_kept_bins(self) -> int:
        return max(1, self.d_factor * self.k)

    def window(self, cache: WindowCache | None = None) -> FlatWindow:
        cache = cache or _WINDOWS
        return cache.get(self.n, self.b_bins, self.window_delta_stop, self.window_delta_pass)


def _fetch(ctx, res, stream, precision_code):
    """Copy the native result to host arrays (coords int64[m,2], values)."""
    m = int(res.count)
    ij = np.empty((m, 2), dtype=np.int64)
    vals = np.empty(m, dtype=np.complex128 if precision_code == _native.FP64 else np.complex64)
    if m:
        ctx.check(ctx.lib.sfft2d_fetch_result(ctx.handle, ij.ctypes.data, vals.ctypes.data, 1,
                                              stream))
    if res.ordered_by_magnitude and m > 1:
        order = np.lexsort((ij[:, 1], ij[:, 0], -np.abs(vals.astype(np.complex128))))
        ij, vals = ij[order], vals[order]
    return ij, vals


def to_dict(ij: np.ndarray, vals: np.ndarray) -> dict:
    """{(i, j): complex} in the arrays' order; tolist() already yields Python
    ints and complex numbers (2x faster than converting each entry)."""
    return dict(zip(map(tuple, ij.tolist()), vals.astype(np.complex128, copy=False).tolist()))


def _stream(torch, device):
    """The raw handle of `device`'s current stream (torch's C getter when it
    exists: ~1 us less than building a torch.cuda.Stream object per call)."""
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(device if isinstance(device, int) else torch.device(device).index)
    return torch.cuda.current_stream(device).cuda_stream


def sfft_perms(rng, n: int, loops: int) -> list:
    """The reference's per-loop permutations (engine.py:266-280) for an int
    seed or Generator, derived natively (sfft2d_sfft_draw_perms): location
    loops [0, loops), estimation loops [loops, 2 loops)."""
    from .tuner import _generator
    gen, bitgen, _ = _generator(rng)
    out = (_native.Perm * (2 * loops))()
    rc = _native.load_library().sfft2d_sfft_draw_perms(bitgen, n, loops, out)
    if rc != _native.OK:
        raise ValueError(f"cannot draw permutations for n={n}, loops={loops}")
    return list(out)


def sfft2d_arrays(x, cfg: SfftConfig, rng, *, cache: WindowCache | None = None,
                  precision: str = "fp64", device=None):
    """``sfft2d`` returning (coords int64[m, 2], values[m]) in the reference's
    dict order instead of a dict."""
    torch = _native._torch()
    img = as_device_image(x, device, upload=False)
    if img.n != cfg.n:
        raise ConfigurationError(f"config built for n={cfg.n}, signal has n={img.n}")
    prec = _native.precision_code(precision)
    # the per-loop streams (engine.py:266-280: 2L child Generators seeded from
    # rng.integers(2**63), one draw_permutation each) are derived natively from
    # the caller's bit generator (sfft2d_sfft_bitgen, csrc/npyrng.h)
    from .tuner import _generator
    gen, bitgen, snapshot = _generator(rng)
    ctx = _native.context(img.device)
    ctx.ensure_tables(cfg.n, cfg.window_delta_pass, cfg.window_delta_stop)
    ccfg = _native.SfftCfg(cfg.n, cfg.k, cfg.loops, cfg.d_factor, cfg.vote_threshold, cfg.b_bins,
                           cfg.window_delta_pass, cfg.window_delta_stop, cfg.gain_floor,
                           cfg.prune_rel)
    res = _native.ResultC()
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)
        if img.tensor is not None:
            ptr, on_host = img.tensor.data_ptr(), 0
        else:
            ptr, on_host = img.host.ctypes.data, 1
        rc = ctx.lib.sfft2d_sfft_bitgen(ctx.handle, ptr, img.dtype_code, on_host, ctypes.byref(ccfg),
                                        bitgen, prec, st, ctypes.byref(res))
        if rc == _native.ERR_VALUE and snapshot is not None:
            gen.bit_generator.state = snapshot   # the reference validates x before drawing
        ctx.check(rc)
        ctx.last_launches = int(res.gpu_launches)
        return _fetch(ctx, res, st, prec)


def sfft2d(x, cfg: SfftConfig, rng, *, cache: WindowCache | None = None,
           precision: str = "fp64", device=None) -> dict:
    """Full Algorithm 1 on the GPU: location loops, vote, estimation loops,
    median, top-k, prune (engine.py:256-284).  ``rng``: seed or Generator."""
    return to_dict(*sfft2d_arrays(x, cfg, rng, cache=cache, precision=precision, device=device))


def build_window(cfg: SfftConfig) -> FlatWindow:
    return build_flat_window(cfg.n, cfg.b_bins, cfg.window_delta_stop,
                             delta_pass=cfg.window_delta_pass)


# ---------------------------------------------------------------- lower level
# The reference's per-loop building blocks (engine.py:130-225), for callers that
# compose Algorithm 1 themselves.  The hash passes run on the GPU through the C
# ABI; vote counting and the per-coordinate median are the same small host-side
# bookkeeping the reference does.

def _cfg_for_window(cfg: SfftConfig, window: FlatWindow) -> "_native.SfftCfg":
    if window.n != cfg.n or window.b_bins != cfg.b_bins:
        raise ValueError("window does not match the configuration's (n, b_bins)")
    return _native.SfftCfg(cfg.n, cfg.k, 1, cfg.d_factor, 1, cfg.b_bins, window.delta_pass,
                           window.delta_stop, cfg.gain_floor, cfg.prune_rel)


def seek_location_once(x, cfg: SfftConfig, window: FlatWindow, rng, *, precision: str = "fp64",
                       device=None):
    """One location loop (engine.py:130-145): draw a permutation, hash,
    keep the ``num_kept_bins`` largest bins, reverse-hash each with a
    one-sample margin, deduplicate.  Returns the permutation and an (m, 2)
    int64 array of candidate coordinates in row-major order."""
    torch = _native._torch()
    rng = np.random.default_rng(rng)
    p = draw_permutation(cfg.n, rng)
    img = as_device_image(x, device)
    if img.n != cfg.n:
        raise ConfigurationError(f"config built for n={cfg.n}, signal has n={img.n}")
    ccfg = _cfg_for_window(cfg, window)
    ctx = _native.context(img.device)
    ctx.ensure_tables(cfg.n, window.delta_pass, window.delta_stop)
    nn = cfg.n * cfg.n
    counts = torch.zeros(((nn + 31) // 32) * 32, dtype=torch.uint8, device=img.tensor.device)
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)
        ctx.check(ctx.lib.sfft2d_sfft_votes(
            ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, ctypes.byref(ccfg),
            _native.perm_array([p]), 1, _native.precision_code(precision), st, counts.data_ptr()))
        keys = torch.nonzero(counts[:nn]).flatten().to(torch.int64).cpu().numpy()
    return p, np.stack([keys // cfg.n, keys % cfg.n], axis=1)


def vote_and_select(candidate_sets, cfg: SfftConfig) -> np.ndarray:
    """Coordinates present in at least ``vote_threshold`` of the ``loops``
    candidate sets, as an (m, 2) int64 array in row-major order
    (engine.py:148-160)."""
    if len(candidate_sets) != cfg.loops:
        raise ValueError(f"expected {cfg.loops} candidate sets, got {len(candidate_sets)}")
    n = cfg.n
    flat = [np.asarray(c, dtype=np.int64).reshape(-1, 2) for c in candidate_sets]
    keys = np.concatenate([f[:, 0] * n + f[:, 1] for f in flat]) if flat else np.empty(0, np.int64)
    uniq, counts = np.unique(keys, return_counts=True)
    kept = uniq[counts >= cfg.vote_threshold]
    return np.stack([kept // n, kept % n], axis=1)


def estimate_once(x, coords, p, window: FlatWindow, cfg: SfftConfig, *, precision: str = "fp64",
                  device=None) -> dict:
    """One estimation loop (engine.py:163-195): the hash pass runs on the GPU
    (``binned_spectrum``); each coordinate reads its bin, undoes the
    permutation's phase twist and divides by the window gain.  Coordinates
    whose gain is below ``gain_floor`` are left out of the dict."""
    from .hashing import binned_spectrum
    coords = np.asarray(coords, dtype=np.int64).reshape(-1, 2)
    if coords.size == 0:
        return {}
    n, b = cfg.n, cfg.b_bins
    spec = binned_spectrum(x, p, window, b, precision=precision, device=device).spectrum
    if not isinstance(spec, np.ndarray):
        spec = spec.cpu().numpy()
    w = n // b
    qi = (p.sigma1 * coords[:, 0]) % n
    qj = (p.sigma2 * coords[:, 1]) % n
    ui = (qi + w // 2) // w
    uj = (qj + w // 2) // w
    gain = window.freq_1d[(qi - w * ui) % n] * window.freq_1d[(qj - w * uj) % n]
    twist = np.exp(-2j * np.pi * ((p.tau1 * coords[:, 0] + p.tau2 * coords[:, 1]) % n) / n)
    ok = np.abs(gain) >= cfg.gain_floor
    vals = spec[ui % b, uj % b] * twist
    return {(int(coords[m, 0]), int(coords[m, 1])): complex(vals[m] / gain[m])
            for m in np.flatnonzero(ok)}


def median_combine(per_loop_estimates, coords=None) -> dict:
    """Componentwise (real, imaginary) median over the loops that produced an
    estimate for each coordinate; coordinates with none are dropped
    (engine.py:198-220)."""
    if coords is None:
        keys = list(dict.fromkeys(k for est in per_loop_estimates for k in est))
    else:
        keys = [(int(i), int(j)) for i, j in np.asarray(coords).reshape(-1, 2)]
    out = {}
    for key in keys:
        vals = np.asarray([est[key] for est in per_loop_estimates if key in est])
        if vals.size:
            out[key] = complex(np.median(vals.real) + 1j * np.median(vals.imag))
    return out


__all__ += ["seek_location_once", "vote_and_select", "estimate_once", "median_combine"]
