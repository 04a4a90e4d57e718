"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain numpy restatement of the reference's hot path (2D SFFT, Algorithm 1,
and ATSFFT, Algorithm 2) used as the parity checker for the sm_100a path.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module; the product package never
does (it fails loudly without its CUDA library instead).

Pinning: ``oracle/make_golden.py`` runs the real reference
(``/root/reference/pkg/src/sfft2d``, importable only in the dev container) on
seeded inputs and writes ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this module against every one of those fixtures (windows, binned
spectra, local maxima, tuner trajectories, votes and recovered spectra).

Every function cites the reference ``file:line`` it restates.  All arithmetic
is float64 / complex128 like the reference (``corefft.py:44``).  Dense FFTs
restate the reference's iterative radix-2 DIT (``corefft.py:54-109``:
bit-reversed gather, per-stage twiddles exp(-2 pi i j/m), butterflies in the
same order), so the oracle's float64 results are bit-identical to the
reference's and decisions taken on roundoff-level near-ties (top-2k among
leakage bins, local maxima of noise-free grids) agree with it exactly.
``FAST = True`` swaps in numpy's pocketfft (CPU timing baseline only).
"""

from __future__ import annotations

import math
from statistics import NormalDist
from typing import NamedTuple

import numpy as np


FAST = False


def _bitrev_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def radix2(a: np.ndarray, inverse: bool = False) -> np.ndarray:
    """Unnormalised radix-2 DIT along the last axis (corefft.py:77-98)."""
    n = a.shape[-1]
    if n == 1:
        return a.copy()
    if FAST:
        return np.fft.ifft(a, axis=-1) * n if inverse else np.fft.fft(a, axis=-1)
    out = np.ascontiguousarray(a[..., _bitrev_perm(n)])
    rows = out.reshape(-1, n)
    m = 2
    while m <= n:
        h = m // 2
        w = np.exp(-2j * np.pi * np.arange(h) / m)
        if inverse:
            w = np.conj(w)
        blk = rows.reshape(rows.shape[0], n // m, m)
        upper = blk[..., h:] * w
        lower = blk[..., :h]
        blk[..., h:] = lower - upper
        blk[..., :h] = lower + upper
        m *= 2
    return out


def fft2(a: np.ndarray) -> np.ndarray:
    """Forward unscaled 2D DFT, rows then columns (corefft.py:101-109)."""
    y = radix2(np.asarray(a, dtype=np.complex128))
    return np.ascontiguousarray(radix2(y.T).T)


class OracleConfigError(ValueError):
    """Mirror of ``engine.ConfigurationError`` (engine.py:45-46)."""


def _pow2(v: int) -> bool:
    return v >= 1 and (v & (v - 1)) == 0


def as_c128(x) -> np.ndarray:
    """Validation + upcast of ``corefft.as_complex_matrix`` (corefft.py:38-51)."""
    a = np.asarray(x, dtype=np.complex128)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {a.shape}")
    if not _pow2(a.shape[0]):
        raise ValueError(f"side {a.shape[0]} is not a power of 2")
    if not np.isfinite(a).all():
        raise ValueError("matrix contains NaN or Inf")
    return a


# --------------------------------------------------------------------------
# permutations (hashing.py:45-80)
# --------------------------------------------------------------------------
class Perm(NamedTuple):
    n: int
    s1: int
    s2: int
    t1: int
    t2: int
    s1i: int
    s2i: int


def make_perm(n: int, s1: int, s2: int, t1: int, t2: int) -> Perm:
    """``PermutationParams`` incl. cached inverses (hashing.py:45-69)."""
    if s1 % 2 == 0 or s2 % 2 == 0:
        raise ValueError("sigma1 and sigma2 must be odd")
    inv = (lambda s: pow(s % n, -1, n)) if n > 1 else (lambda s: 0)
    return Perm(n, s1, s2, t1, t2, inv(s1), inv(s2))


def draw_perm(n: int, gen: np.random.Generator) -> Perm:
    """Four scalar draws in the reference order (hashing.py:72-80)."""
    if n > 1:
        s1 = 2 * int(gen.integers(0, n // 2)) + 1
        s2 = 2 * int(gen.integers(0, n // 2)) + 1
    else:
        s1 = s2 = 1
    t1 = int(gen.integers(0, n))
    t2 = int(gen.integers(0, n))
    return make_perm(n, s1, s2, t1, t2)


# --------------------------------------------------------------------------
# flat window (hashing.py:138-261)
# --------------------------------------------------------------------------
class Window(NamedTuple):
    n: int
    b: int
    support: int
    half: int
    pass_hw: int
    space: np.ndarray     # f64[n]
    freq: np.ndarray      # f64[n]


def _upper_q(p: float) -> float:
    return -NormalDist().inv_cdf(p)


def window(n: int, b: int, dstop: float = 1e-8, dpass: float = 1e-6) -> Window:
    """Gaussian-smoothed boxcar window (hashing.py:138-225; all-pass at b == n, :228-246)."""
    if not _pow2(n) or not _pow2(b):
        raise ValueError("n and b must be powers of 2")
    if b > n or n % b:
        raise ValueError(f"bin count {b} must divide side {n}")
    if not (0.0 < dpass < 0.5 and 0.0 < dstop < 0.5):
        raise ValueError("tolerances must lie in (0, 0.5)")
    if b == n:
        delta = np.zeros(n)
        delta[0] = 1.0
        return Window(n, n, n, n // 2, 0, np.ones(n), delta)
    w = n // b
    half_pass = w // 2
    zp, zs = _upper_q(dpass / 8), _upper_q(dstop / 4)
    width = (w - half_pass) / (zp + zs)
    edge = half_pass + zp * width
    dist = np.minimum(np.arange(n), n - np.arange(n)).astype(float)
    cdf = np.vectorize(lambda z: 0.5 * math.erfc(-z / math.sqrt(2.0)), otypes=[float])
    resp = cdf((edge - dist) / width) + cdf((edge + dist) / width) - 1.0
    proto = radix2(resp.astype(np.complex128), inverse=True).real / n
    proto = 0.5 * (proto + np.roll(proto[::-1], 1))
    budget = min(dpass / 8, dstop / 4) * resp[0]
    # tail(h) = sum of |proto| over samples farther than h, accumulated from the
    # farthest sample inwards in stable-by-distance order (hashing.py:188-198)
    by_dist = np.argsort(dist, kind="stable")
    mags_sorted = np.abs(proto)[by_dist]
    tails = np.append(np.cumsum(mags_sorted[::-1])[::-1], 0.0)
    dist_sorted = dist[by_dist]
    half = n // 2
    for h in range(n // 2 + 1):
        if tails[np.searchsorted(dist_sorted, h + 0.5)] <= budget:
            half = h
            break
    support = min(2 * half + 1, n)
    space = proto.copy() if support >= n else np.where(dist <= half, proto, 0.0)
    space *= n / space.sum()
    freq = radix2(space.astype(np.complex128)).real / n
    freq = freq / freq[0]
    freq = 0.5 * (freq + np.roll(freq[::-1], 1))
    return Window(n, b, support, half if support < n else n // 2, half_pass, space, freq)


_WIN: dict = {}


def cached_window(n, b, dstop, dpass) -> Window:
    key = (n, b, dpass, dstop)
    if key not in _WIN:
        _WIN[key] = window(n, b, dstop, dpass)
    return _WIN[key]


# --------------------------------------------------------------------------
# hash pass (hashing.py:308-337) and coordinate maps (:340-395)
# --------------------------------------------------------------------------
def bucket_spectrum(a: np.ndarray, p: Perm, win: Window, b: int) -> np.ndarray:
    """Gather the permuted support, window it, fold it to b x b, 2D DFT."""
    n = a.shape[0]
    if win.n != n or win.b != b:
        raise ValueError("window does not match the requested (n, b)")
    if win.support >= n:
        offs = np.arange(n)
    else:
        h = win.half
        offs = np.arange(-b * ((h + b - 1) // b), b * ((h + b) // b))
    pos = offs % n
    rsel = (p.s1 * pos + p.t1) % n
    csel = (p.s2 * pos + p.t2) % n
    g = win.space[pos]
    blk = a[np.ix_(rsel, csel)] * g[:, None] * g[None, :]
    m = offs.size
    folded = blk.reshape(m // b, b, m // b, b).sum(axis=(0, 2))
    return fft2(folded)


def axis_hash(q, n: int, b: int):
    """(bin, signed offset) of permuted frequencies (hashing.py:340-345)."""
    w = n // b
    u = (np.asarray(q) + w // 2) // w
    return u % b, np.asarray(q) - w * u


def preimage_axis(bins: np.ndarray, sinv: int, n: int, b: int, expand: int) -> np.ndarray:
    """Vectorised ``_unhash_axis`` for many bins at once (hashing.py:368-376):
    row r holds the preimage frequencies of bins[r]."""
    w = n // b
    bins = np.asarray(bins, dtype=np.int64).reshape(-1)
    if w == 1 and expand == 0:
        t = bins[:, None]
    else:
        length = min(w + 2 * expand, n)
        lo = bins * w - w // 2 - expand
        t = (lo[:, None] + np.arange(length)[None, :]) % n
    return (sinv * t) % n


def preimage_keys(bi, bj, p: Perm, n: int, b: int, expand: int) -> np.ndarray:
    """Flat keys i*n+j of every bin's preimage grid, bin-major then i-major
    (the order ``_unhash_grid`` emits, hashing.py:379-386)."""
    ii = preimage_axis(bi, p.s1i, n, b, expand)
    jj = preimage_axis(bj, p.s2i, n, b, expand)
    return (ii[:, :, None] * n + jj[:, None, :]).reshape(-1)


# --------------------------------------------------------------------------
# Algorithm 1 (engine.py)
# --------------------------------------------------------------------------
def nearest_pow2(v: float) -> int:
    """engine.py:49-52 (ties go to the lower power)."""
    lo = 1 << max(int(math.floor(math.log2(v))), 0) if v >= 1 else 1
    return lo if (v - lo) <= (2 * lo - v) else 2 * lo


def default_bins(n: int, k: int) -> int:
    """engine.py:55-66."""
    k = max(k, 1)
    return max(4, min(nearest_pow2(math.sqrt(min(n, 256) * k)), n))


class SfftParams(NamedTuple):
    n: int
    k: int
    loops: int
    d_factor: int
    threshold: int
    b: int
    dpass: float
    dstop: float
    gain_floor: float
    prune_rel: float

    @property
    def kept(self) -> int:
        return max(1, self.d_factor * self.k)


def sfft_params(n, k, loops=8, d_factor=2, vote_threshold=None, b_bins=None, dpass=1e-3,
                dstop=1e-8, gain_floor=1e-6, prune_rel=1e-3) -> SfftParams:
    """``SfftConfig.__post_init__`` validation and defaults (engine.py:69-113)."""
    if not _pow2(n):
        raise OracleConfigError(f"side {n} is not a power of 2")
    if k < 0 or k > n * n:
        raise OracleConfigError("sparsity out of range")
    if loops < 1:
        raise OracleConfigError("loops must be >= 1")
    b = default_bins(n, k) if b_bins is None else b_bins
    if not _pow2(b) or b > n or n % b:
        raise OracleConfigError(f"bin count {b} must be a power of 2 dividing {n}")
    thr = (loops + 1) // 2 if vote_threshold is None else vote_threshold
    if not 1 <= thr <= loops:
        raise OracleConfigError("vote_threshold out of range")
    if max(1, d_factor * k) > b * b:
        raise OracleConfigError("d_factor*k exceeds the bin budget")
    return SfftParams(n, k, loops, d_factor, thr, b, dpass, dstop, gain_floor, prune_rel)


def top_bins(spec: np.ndarray, num: int) -> np.ndarray:
    """engine.py:122-127: stable descending magnitude order, first ``num``."""
    return np.argsort(-np.abs(spec).ravel(), kind="stable")[:num]


def location_loop(a, cfg: SfftParams, win: Window, p: Perm) -> np.ndarray:
    """One location loop with per-loop dedup (engine.py:130-145); returns sorted keys."""
    spec = bucket_spectrum(a, p, win, cfg.b)
    flat = top_bins(spec, cfg.kept)
    keys = preimage_keys(flat // cfg.b, flat % cfg.b, p, cfg.n, cfg.b, expand=1)
    return np.unique(keys)


def vote(key_sets, threshold: int) -> np.ndarray:
    """engine.py:148-160: keys seen in >= threshold sets (sorted)."""
    allk = np.concatenate([np.asarray(s, dtype=np.int64) for s in key_sets]) if key_sets else \
        np.empty(0, np.int64)
    uniq, cnt = np.unique(allk, return_counts=True)
    return uniq[cnt >= threshold]


def estimate(a, coords: np.ndarray, p: Perm, win: Window, b: int, gain_floor: float):
    """engine.py:163-177: per-coordinate value and usability for one loop."""
    n = a.shape[0]
    spec = bucket_spectrum(a, p, win, b)
    w = n // b
    i, j = coords[:, 0], coords[:, 1]
    qi, qj = (p.s1 * i) % n, (p.s2 * j) % n
    ui, uj = (qi + w // 2) // w, (qj + w // 2) // w
    gain = win.freq[(qi - w * ui) % n] * win.freq[(qj - w * uj) % n]
    twist = np.exp(-2j * np.pi * ((p.t1 * i + p.t2 * j) % n) / n)
    raw = spec[ui % b, uj % b] * twist
    ok = np.abs(gain) >= gain_floor
    return np.where(ok, raw / np.where(ok, gain, 1.0), 0.0), ok


def median_pick(coords, vals_list, ok_list, k: int, prune_rel: float):
    """engine.py:228-253. Returns (coords int64[m,2], values c128[m]) in the
    reference's dict insertion order."""
    vals = np.stack(vals_list)
    ok = np.stack(ok_list)
    alive = ok.sum(axis=0) > 0
    if not alive.any():
        return np.empty((0, 2), np.int64), np.empty(0, np.complex128)
    data = np.where(ok, vals, np.nan)[:, alive]
    med = np.nanmedian(data.real, axis=0) + 1j * np.nanmedian(data.imag, axis=0)
    cs = coords[alive]
    mag = np.abs(med)
    if mag.size > k:
        sel = np.lexsort((cs[:, 1], cs[:, 0], -mag))[:k]
        cs, med, mag = cs[sel], med[sel], mag[sel]
    if prune_rel > 0 and mag.size:
        keep = mag >= prune_rel * mag.max()
        cs, med = cs[keep], med[keep]
    return cs, med


def sfft(x, cfg: SfftParams, seed, *, return_trace: bool = False):
    """Algorithm 1 end to end (engine.py:256-284). Returns (coords, values)."""
    a = as_c128(x)
    if a.shape[0] != cfg.n:
        raise OracleConfigError("config built for another side")
    gen = np.random.default_rng(seed)
    win = cached_window(cfg.n, cfg.b, cfg.dstop, cfg.dpass)
    kids = [np.random.default_rng(int(gen.integers(2**63))) for _ in range(2 * cfg.loops)]
    loc_perms = [draw_perm(cfg.n, kids[i]) for i in range(cfg.loops)]
    sets = [location_loop(a, cfg, win, p) for p in loc_perms]
    keys = vote(sets, cfg.threshold)
    trace = {"loc_perms": loc_perms, "keys": keys}
    if keys.size == 0:
        out = (np.empty((0, 2), np.int64), np.empty(0, np.complex128))
        return (out, trace) if return_trace else out
    coords = np.stack([keys // cfg.n, keys % cfg.n], axis=1)
    vl, ol = [], []
    est_perms = [draw_perm(cfg.n, kids[cfg.loops + i]) for i in range(cfg.loops)]
    for p in est_perms:
        v, o = estimate(a, coords, p, win, cfg.b, cfg.gain_floor)
        vl.append(v)
        ol.append(o)
    trace["est_perms"] = est_perms
    out = median_pick(coords, vl, ol, cfg.k, cfg.prune_rel)
    return (out, trace) if return_trace else out


# --------------------------------------------------------------------------
# Algorithm 2 (tuner.py)
# --------------------------------------------------------------------------
class TunerParams(NamedTuple):
    b0: int = 16
    eps1: float = 0.5
    eps2: float = 1.0
    delta1: float = 0.02
    delta2: float = 0.05
    max_iters: int | None = None
    mag_floor: float = 1e-3
    dpass: float = 1e-3
    dstop: float = 1e-8
    gain_floor: float = 1e-6
    prune_rel: float = 1e-3

    def iters(self, n: int) -> int:
        """tuner.py:75-78."""
        return self.max_iters if self.max_iters is not None else 2 * max(int(math.log2(n)), 1)


def local_maxima(spec: np.ndarray, floor_rel: float):
    """tuner.py:97-118: strict 8-neighbour toroidal maxima above the floor,
    row-major coordinates."""
    s = np.asarray(spec)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise ValueError("expected a square bin grid")
    if s.shape[0] < 4:
        raise ValueError("bin grid must be at least 4x4")
    m = np.abs(s)
    top = m.max()
    keep = m >= floor_rel * top if top > 0 else np.zeros(m.shape, bool)
    for du in (-1, 0, 1):
        for dv in (-1, 0, 1):
            if du or dv:
                keep &= m > np.roll(m, (du, dv), axis=(0, 1))
    where = np.argwhere(keep)
    return int(keep.sum()), where


def next_bins(b: int, r: float, cfg: TunerParams, n: int) -> int:
    """tuner.py:121-130."""
    if r < cfg.delta1:
        v = b * cfg.eps1
    elif r < cfg.delta2:
        v = float(b)
    else:
        v = b * (1.0 + cfg.eps2)
    return max(4, min(nearest_pow2(v), n))


def detect(a: np.ndarray, cfg: TunerParams, gen: np.random.Generator):
    """tuner.py:142-241. Returns (state dict, (coords, tallies), perms used)."""
    n = a.shape[0]
    iters = cfg.iters(n)
    b = max(4, min(cfg.b0, n))
    hist: list = []
    converged = False
    seen: dict = {}
    moved = False
    chunks: list = []
    vote_passes = 0
    last = None
    prev = None
    budget = max(n * n // 8, 1 << 16)
    perms: list = []

    def one_pass(bb):
        nonlocal vote_passes, last
        win = cached_window(n, bb, cfg.dstop, cfg.dpass)
        p = draw_perm(n, gen)
        perms.append(p)
        cnt, mx = local_maxima(bucket_spectrum(a, p, win, bb), cfg.mag_floor)
        last = (p, mx, bb)
        w = n // bb
        if cnt > 0 and cnt * (w + 2) ** 2 <= budget:
            vote_passes += 1
            chunks.append(preimage_keys(mx[:, 0], mx[:, 1], p, n, bb, expand=1))
        return cnt

    for _ in range(iters):
        cnt = one_pass(b)
        if prev is None:
            r = None
        elif prev == 0 and cnt == 0:
            hist.append((b, cnt, 0.0))
            converged = True
            break
        else:
            r = math.inf if prev == 0 else abs(1.0 - cnt / prev)
        hist.append((b, cnt, r))
        if r is not None and cfg.delta1 <= r < cfg.delta2:
            converged = True
            break
        seen[(b, cnt)] = seen.get((b, cnt), 0) + 1
        if seen[(b, cnt)] >= 3 and moved:
            converged = True
            break
        prev = cnt
        if r is not None:
            nb = next_bins(b, r, cfg, n)
            moved = moved or nb != b
            b = nb

    counts = [c for _, c, _ in hist]
    if counts and max(counts) > 0:
        top = max(bb for bb, _, _ in hist)
        for bc in (2 * top, 4 * top):
            if bc <= n:
                cnt = one_pass(bc)
                hist.append((bc, cnt, None))
                counts.append(cnt)
    det_k = max(counts) if counts else 0
    b_detect = max((bb for bb, _, _ in hist), default=b)
    b_est = default_bins(n, det_k)
    if not chunks and last is not None and det_k > 0:
        p, mx, bb = last
        chunks.append(preimage_keys(mx[:, 0], mx[:, 1], p, n, bb, expand=1))
        vote_passes = 1
    if chunks:
        uniq, tal = np.unique(np.concatenate(chunks), return_counts=True)
        votes = (np.stack([uniq // n, uniq % n], axis=1), tal)
    else:
        votes = (np.empty((0, 2), np.int64), np.empty(0, np.int64))
    state = dict(history=hist, converged=converged, detected_k=det_k, b_detect=b_detect,
                 b_estimate=b_est, vote_passes=vote_passes)
    return state, votes, perms


def atsfft(x, cfg: TunerParams, est_loops: int, seed, *, return_trace: bool = False):
    """tuner.py:244-282. Returns ((coords, values), state)."""
    a = as_c128(x)
    n = a.shape[0]
    gen = np.random.default_rng(seed)
    state, (vc, vt), perms = detect(a, cfg, gen)
    trace = {"perms": perms, "votes": (vc, vt)}
    empty = (np.empty((0, 2), np.int64), np.empty(0, np.complex128))
    if state["detected_k"] == 0 or vc.shape[0] == 0:
        return (empty, state, trace) if return_trace else (empty, state)
    thr = (max(state["vote_passes"], 1) + 1) // 2
    coords = vc[vt >= thr]
    if coords.shape[0] == 0:
        return (empty, state, trace) if return_trace else (empty, state)
    ecfg = sfft_params(n, state["detected_k"], loops=max(est_loops, 1), b_bins=state["b_estimate"],
                       dpass=cfg.dpass, dstop=cfg.dstop, gain_floor=cfg.gain_floor,
                       prune_rel=cfg.prune_rel)
    win = cached_window(n, ecfg.b, ecfg.dstop, ecfg.dpass)
    vl, ol, eperms = [], [], []
    for _ in range(ecfg.loops):
        p = draw_perm(n, gen)
        eperms.append(p)
        v, o = estimate(a, coords, p, win, ecfg.b, ecfg.gain_floor)
        vl.append(v)
        ol.append(o)
    trace["est_perms"] = eperms
    trace["coords"] = coords
    out = median_pick(coords, vl, ol, state["detected_k"], cfg.prune_rel)
    return (out, state, trace) if return_trace else (out, state)


def as_dict(out) -> dict:
    cs, vs = out
    return {(int(i), int(j)): complex(v) for (i, j), v in zip(cs, vs)}
