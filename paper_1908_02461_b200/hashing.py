"""Hash front end: permutations, flat windows (host setup) and the GPU
``binned_spectrum`` — mirror of ``/root/reference/pkg/src/sfft2d/hashing.py``.

Host side (setup, like an FFT plan): permutation draws from the caller's numpy
Generator in the reference's exact order, and the flat window
(``build_flat_window``) computed with the reference's formulas in float64.
The window tables for every bin count of a side N are registered once with the
native context (device-resident), so a transform never rebuilds them.

Device side: ``binned_spectrum`` is the fused permute/window/fold + bucket FFT
kernel pair (``csrc/fold.cuh`` + ``csrc/fft.cuh``).
"""

from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field
from statistics import NormalDist

import numpy as np

from . import _native
from ._tensors import as_device_image, to_numpy_complex

__all__ = [
    "PermutationParams", "FlatWindow", "BinGrid", "draw_permutation", "identity_permutation",
    "build_flat_window", "all_pass_window", "WindowCache", "binned_spectrum", "hash_coord",
    "offset_coord", "unhash_bin", "mod_inverse",
]


def is_power_of_two(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def mod_inverse(a: int, n: int) -> int:
    """Inverse of odd ``a`` modulo the power of two ``n`` (corefft.py:135-146)."""
    if not is_power_of_two(n):
        raise ValueError(f"modulus {n} is not a power of 2")
    a = a % n
    if n > 1 and a % 2 == 0:
        raise ValueError(f"{a} is even and has no inverse modulo {n}")
    return pow(a, -1, n)


@dataclass(frozen=True)
class PermutationParams:
    """Spectrum permutation (hashing.py:45-69): (i, j) -> (sigma1 i, sigma2 j) mod n."""

    n: int
    sigma1: int
    sigma2: int
    tau1: int
    tau2: int
    sigma1_inv: int = field(default=-1)
    sigma2_inv: int = field(default=-1)

    def __post_init__(self):
        if self.sigma1 % 2 == 0 or self.sigma2 % 2 == 0:
            raise ValueError("sigma1 and sigma2 must be odd")
        if self.sigma1_inv < 0:
            object.__setattr__(self, "sigma1_inv", mod_inverse(self.sigma1, self.n))
        if self.sigma2_inv < 0:
            object.__setattr__(self, "sigma2_inv", mod_inverse(self.sigma2, self.n))


def draw_permutation(n: int, rng: np.random.Generator) -> PermutationParams:
    """Four scalar draws, sigma1, sigma2 odd then tau1, tau2 (hashing.py:72-80)."""
    if not is_power_of_two(n):
        raise ValueError(f"side {n} is not a power of 2")
    if n > 1:
        s1 = 2 * int(rng.integers(0, n // 2)) + 1
        s2 = 2 * int(rng.integers(0, n // 2)) + 1
    else:
        s1 = s2 = 1
    t1 = int(rng.integers(0, n))
    t2 = int(rng.integers(0, n))
    return PermutationParams(n, s1, s2, t1, t2)


def identity_permutation(n: int) -> PermutationParams:
    return PermutationParams(n, 1, 1, 0, 0)


@dataclass(frozen=True)
class FlatWindow:
    """Separable flat window (hashing.py:96-135)."""

    n: int
    b_bins: int
    support_w: int
    half_support: int
    pass_halfwidth: int
    delta_pass: float
    delta_stop: float
    space_1d: np.ndarray
    freq_1d: np.ndarray

    def gain(self, off_i, off_j):
        g = self.freq_1d
        return g[np.asarray(off_i) % self.n] * g[np.asarray(off_j) % self.n]

    def support_offsets(self) -> np.ndarray:
        if self.support_w >= self.n:
            return np.arange(self.n)
        return np.arange(-self.half_support, self.half_support + 1)

    def space_block(self) -> np.ndarray:
        g = self.space_1d[self.support_offsets() % self.n]
        return np.outer(g, g)

    def freq_response_2d(self) -> np.ndarray:
        return np.outer(self.freq_1d, self.freq_1d)


def all_pass_window(n: int) -> FlatWindow:
    """Identity filter for b == n (hashing.py:228-246)."""
    freq = np.zeros(n)
    freq[0] = 1.0
    return FlatWindow(n, n, n, n // 2, 0, 1e-12, 1e-12, np.ones(n), freq)


_std_normal = NormalDist()


def _gauss_cdf(z: np.ndarray) -> np.ndarray:
    # elementwise 0.5*erfc(-z/sqrt2) with math.erfc, as the reference (hashing.py:92-93)
    root2 = math.sqrt(2.0)
    return np.fromiter((0.5 * math.erfc(-v / root2) for v in z), dtype=float, count=z.size)


def build_flat_window(n: int, b: int, delta_stop: float = 1e-8, *, delta_pass: float = 1e-6,
                      max_support: int | None = None) -> FlatWindow:
    """Boxcar (width n/b) smoothed by a Gaussian, truncated to the shortest
    support whose discarded tail stays within budget (hashing.py:138-225)."""
    if not is_power_of_two(n) or not is_power_of_two(b):
        raise ValueError("n and b must be powers of 2")
    if b > n or n % b != 0:
        raise ValueError(f"bin count {b} must divide side {n}")
    if not (0.0 < delta_pass < 0.5 and 0.0 < delta_stop < 0.5):
        raise ValueError("tolerances must lie in (0, 0.5)")
    if b == n:
        w = all_pass_window(n)
        return FlatWindow(n, n, n, n // 2, 0, delta_pass, delta_stop, w.space_1d, w.freq_1d)
    w = n // b
    p = w // 2
    z_pass = -_std_normal.inv_cdf(delta_pass / 8)
    z_stop = -_std_normal.inv_cdf(delta_stop / 4)
    sigma_f = (w - p) / (z_pass + z_stop)
    beta = p + z_pass * sigma_f
    dist = np.minimum(np.arange(n), n - np.arange(n)).astype(float)
    gamma = _gauss_cdf((beta - dist) / sigma_f) + _gauss_cdf((beta + dist) / sigma_f) - 1.0
    g_full = np.fft.ifft(gamma.astype(np.complex128)).real
    g_full = 0.5 * (g_full + np.roll(g_full[::-1], 1))
    eps_t = min(delta_pass / 8, delta_stop / 4) * gamma[0]
    order = np.argsort(dist, kind="stable")
    sorted_dist = dist[order]
    suffix = np.concatenate([np.cumsum(np.abs(g_full)[order][::-1])[::-1], [0.0]])
    # tail(h) is non-increasing in h: binary search for the first h within budget
    lo, hi = 0, n // 2
    if suffix[np.searchsorted(sorted_dist, hi + 0.5)] > eps_t:
        half = n // 2
    else:
        while lo < hi:
            mid = (lo + hi) // 2
            if suffix[np.searchsorted(sorted_dist, mid + 0.5)] <= eps_t:
                hi = mid
            else:
                lo = mid + 1
        half = lo
    support_w = min(2 * half + 1, n)
    if max_support is not None and support_w > max_support:
        raise ValueError(
            f"tolerances need support {support_w} > budget {max_support} at n={n}, b={b}")
    g1 = g_full.copy() if support_w >= n else np.where(dist <= half, g_full, 0.0)
    g1 *= n / g1.sum()
    ghat = np.fft.fft(g1.astype(np.complex128)).real / n
    ghat = ghat / ghat[0]
    ghat = 0.5 * (ghat + np.roll(ghat[::-1], 1))
    return FlatWindow(n, b, support_w, half if support_w < n else n // 2, p, delta_pass,
                      delta_stop, g1, ghat)


class WindowCache:
    """Memoizes windows per (n, b, delta_pass, delta_stop) (hashing.py:249-261)."""

    def __init__(self):
        self._built: dict = {}

    def get(self, n, b, delta_stop=1e-8, delta_pass=1e-6) -> FlatWindow:
        key = (n, b, delta_pass, delta_stop)
        win = self._built.get(key)
        if win is None:
            win = build_flat_window(n, b, delta_stop, delta_pass=delta_pass)
            self._built[key] = win
        return win


_HOST_WINDOWS = WindowCache()


@functools.lru_cache(maxsize=64)
def host_tables(n: int, delta_pass: float, delta_stop: float):
    """float64 tables registered with the native context: space/freq rows for
    every B = 2^0..n (rows B < 4 unused) and the twiddles exp(-2 pi i k / n)."""
    lg = n.bit_length() - 1
    space = np.zeros((lg + 1, n))
    freq = np.zeros((lg + 1, n))
    b = 4
    while b <= n:
        win = _HOST_WINDOWS.get(n, b, delta_stop, delta_pass)
        space[b.bit_length() - 1] = win.space_1d
        freq[b.bit_length() - 1] = win.freq_1d
        b *= 2
    # same expression as the reference's phase factors (engine.py:173)
    tw = np.exp(-2j * np.pi * np.arange(n) / n)
    tw = np.ascontiguousarray(tw).view(np.float64)
    return np.ascontiguousarray(space), np.ascontiguousarray(freq), tw


def check_window(window: FlatWindow) -> None:
    """The device applies the registered window tables of (n, delta_pass,
    delta_stop), i.e. exactly build_flat_window's weights (all_pass_window's
    at B = n).  A FlatWindow with any other weights would silently get a
    different window than the reference applies (hashing.py:330), so it is
    rejected."""
    want = (all_pass_window(window.n) if window.b_bins == window.n else
            _HOST_WINDOWS.get(window.n, window.b_bins, window.delta_stop, window.delta_pass))
    if window is want:
        return
    if not (np.array_equal(np.asarray(window.space_1d), want.space_1d) and
            np.array_equal(np.asarray(window.freq_1d), want.freq_1d)):
        raise ValueError("window weights differ from build_flat_window(n, b, delta_stop, "
                         "delta_pass=...): only the library's flat windows are supported")


@dataclass(frozen=True)
class BinGrid:
    """DFT of the permuted, filtered, folded signal (hashing.py:300-305)."""

    b_bins: int
    spectrum: object  # numpy array (numpy input) or torch CUDA tensor (tensor input)


def binned_spectrum(x, p: PermutationParams | list, window: FlatWindow, b: int, *,
                    precision: str = "fp64", device=None) -> BinGrid:
    """Fused gather/window/fold/B x B FFT on the GPU (hashing.py:308-337).

    ``p`` may be one permutation or a list of them (hash loops sharing one read
    of the image; the result then has a leading loop axis).
    """
    torch = _native._torch()
    img = as_device_image(x, device)
    n = img.n
    if window.n != n or b != window.b_bins:
        raise ValueError("window does not match the requested (n, b)")
    check_window(window)
    perms = p if isinstance(p, (list, tuple)) else [p]
    prec = _native.precision_code(precision)
    ctx = _native.context(img.device)
    ctx.ensure_tables(n, window.delta_pass, window.delta_stop)
    cdt = torch.complex128 if prec == _native.FP64 else torch.complex64
    out = torch.empty((len(perms), b, b), dtype=cdt, device=img.tensor.device)
    parr = _native.perm_array(perms)
    with torch.cuda.device(img.device):
        st = torch.cuda.current_stream().cuda_stream
        ctx.check(ctx.lib.sfft2d_binned_spectrum(
            ctx.handle, img.tensor.data_ptr(), img.dtype_code, n, b, parr, len(perms),
            float(window.delta_pass), float(window.delta_stop), prec, out.data_ptr(), st))
    spec = out if isinstance(p, (list, tuple)) else out[0]
    if img.from_numpy:
        spec = to_numpy_complex(spec)
    return BinGrid(b_bins=b, spectrum=spec)


def _hash_axis(q, n: int, b: int):
    w = n // b
    unwrapped = (np.asarray(q) + w // 2) // w
    return unwrapped % b, np.asarray(q) - w * unwrapped


def hash_coord(i, j, p: PermutationParams, n: int, b: int):
    """Bin of frequency (i, j): round-half-up bucketing of the permuted
    frequency (hashing.py:348-355)."""
    bi, _ = _hash_axis((p.sigma1 * np.asarray(i)) % n, n, b)
    bj, _ = _hash_axis((p.sigma2 * np.asarray(j)) % n, n, b)
    if np.isscalar(i) or (isinstance(i, int) and isinstance(j, int)):
        return int(bi), int(bj)
    return bi, bj


def offset_coord(i, j, p: PermutationParams, n: int, b: int):
    """Residual of the permuted frequency from its bin centre (hashing.py:358-365)."""
    _, oi = _hash_axis((p.sigma1 * np.asarray(i)) % n, n, b)
    _, oj = _hash_axis((p.sigma2 * np.asarray(j)) % n, n, b)
    if np.isscalar(i) or (isinstance(i, int) and isinstance(j, int)):
        return int(oi), int(oj)
    return oi, oj


def _unhash_axis(bin_idx: int, sigma_inv: int, n: int, b: int, expand: int = 0) -> np.ndarray:
    w = n // b
    if w == 1 and expand == 0:
        ts = np.array([bin_idx])
    else:
        lo = bin_idx * w - w // 2 - expand
        ts = (lo + np.arange(min(w + 2 * expand, n))) % n
    return (sigma_inv * ts) % n


def unhash_bin(bin_i: int, bin_j: int, p: PermutationParams, n: int, b: int,
               expand: int = 0) -> np.ndarray:
    """All coordinates hashing to (bin_i, bin_j) as an (m, 2) array, i-major
    (hashing.py:379-395)."""
    ii = _unhash_axis(bin_i, p.sigma1_inv, n, b, expand)
    jj = _unhash_axis(bin_j, p.sigma2_inv, n, b, expand)
    out = np.empty((ii.size * jj.size, 2), dtype=np.int64)
    out[:, 0] = np.repeat(ii, jj.size)
    out[:, 1] = np.tile(jj, ii.size)
    return out
