"""Synthetic k-sparse-spectrum workloads and the average-L1 error metric.

The reference ships only a noiseless unit-spike generator
(``/root/reference/pkg/src/sfft2d/signals.py:42-65``).  BASELINE.json's configs
need noise, log-uniform magnitudes and a clustered low-frequency block
(SURVEY.md D3, §8(d) "D-in"), so the workload is defined here, once:

* ``k`` coefficients at distinct (row, col) positions.  A fraction
  ``cluster_frac`` of them is placed in the wrap-around DC block
  ``{-side/2 .. side/2-1}^2 mod n`` (c5), the rest uniformly over the grid.
* magnitude 1 (``"unit"``) or log-uniform in ``mag_range``; phase U[0, 2pi).
* image = inverse 2D DFT of that spectrum with the ``1/n^2`` convention
  (``corefft.py:112-118``), computed with ``np.fft.ifft2``.
* optional complex Gaussian noise with total variance
  ``mean|x_clean|^2 * 10^(-snr_db/10)``, split evenly between re and im.

Everything is drawn from one ``np.random.default_rng(seed)`` stream, so a seed
fully determines the image (same numpy on the dev container and the GPU box).
This is host-side workload tooling, not part of the transform.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass

import numpy as np

__all__ = ["SparseImage", "DeviceSparseImage", "sparse_image", "device_sparse_image", "planted_image", "error_metric", "image_digest",
           "save_signal", "load_signal"]


@dataclass(frozen=True)
class SparseImage:
    n: int
    k: int
    seed: int
    x: np.ndarray                 # (n, n) complex64 / complex128
    rows: np.ndarray              # int64[k]
    cols: np.ndarray              # int64[k]
    coeffs: np.ndarray            # complex128[k]

    @property
    def truth(self) -> dict:
        return {(int(i), int(j)): complex(c) for i, j, c in zip(self.rows, self.cols, self.coeffs)}


def _is_pow2(v: int) -> bool:
    return v >= 1 and (v & (v - 1)) == 0


def _draw_spectrum(rng, n, k, magnitude, mag_range, cluster_frac, cluster_side):
    """Positions (clustered fraction first, then uniform distinct draws),
    phases and magnitudes, in that stream order."""
    n_clu = int(round(cluster_frac * k)) if cluster_frac > 0 else 0
    side = min(cluster_side, n)
    if n_clu > side * side:
        raise ValueError("cluster block too small for the clustered fraction")
    picked: list[int] = []
    if n_clu:
        half = side // 2
        local = rng.choice(side * side, size=n_clu, replace=False)
        ci = (local // side - half) % n
        cj = (local % side - half) % n
        picked.extend((ci * n + cj).tolist())
    taken = set(picked)
    need = k - n_clu
    while need > 0:
        draw = rng.choice(n * n, size=need, replace=False)
        for f in draw.tolist():
            if f not in taken and need > 0:
                taken.add(f)
                picked.append(f)
                need -= 1
    flat = np.asarray(picked, dtype=np.int64)
    rows, cols = flat // n, flat % n
    phases = rng.uniform(0.0, 2.0 * np.pi, size=k)
    if magnitude == "unit":
        mags = np.ones(k)
    elif magnitude == "loguniform":
        lo, hi = np.log(mag_range[0]), np.log(mag_range[1])
        mags = np.exp(rng.uniform(lo, hi, size=k))
    else:
        raise ValueError(f"unknown magnitude law {magnitude!r}")
    coeffs = mags * np.exp(1j * phases)
    return rows, cols, coeffs


def sparse_image(
    n: int,
    k: int,
    seed: int,
    *,
    snr_db: float | None = None,
    magnitude: str = "unit",
    mag_range: tuple[float, float] = (0.1, 10.0),
    cluster_frac: float = 0.0,
    cluster_side: int = 64,
    dtype=np.complex64,
) -> SparseImage:
    """Seeded k-sparse-spectrum image, optionally noisy (see module docstring)."""
    _check_side_k(n, k)
    rng = np.random.default_rng(seed)
    rows, cols, coeffs = _draw_spectrum(rng, n, k, magnitude, mag_range, cluster_frac, cluster_side)
    spec = np.zeros((n, n), dtype=np.complex128)
    spec[rows, cols] = coeffs
    x = np.fft.ifft2(spec)
    del spec
    if snr_db is not None:
        power = float(np.mean(np.abs(x) ** 2))
        sd = np.sqrt(power * 10.0 ** (-snr_db / 10.0) / 2.0)
        x += sd * rng.standard_normal((n, n))
        x += 1j * sd * rng.standard_normal((n, n))
    return SparseImage(n, k, seed, np.ascontiguousarray(x.astype(dtype)), rows, cols, coeffs)


@dataclass(frozen=True)
class DeviceSparseImage:
    n: int
    k: int
    seed: int
    x: object                     # torch.Tensor (n, n) complex64 / complex128 on the device
    rows: np.ndarray
    cols: np.ndarray
    coeffs: np.ndarray
    noise_sd: float
    noise_seed: int

    @property
    def truth(self) -> dict:
        return {(int(i), int(j)): complex(c) for i, j, c in zip(self.rows, self.cols, self.coeffs)}


def _check_side_k(n, k):
    if not _is_pow2(n):
        raise ValueError(f"side {n} is not a power of 2")
    if k < 0 or k > n * n:
        raise ValueError(f"sparsity {k} out of range for side {n}")


def device_sparse_image(
    n: int,
    k: int,
    seed: int,
    *,
    snr_db: float | None = None,
    magnitude: str = "unit",
    mag_range: tuple[float, float] = (0.1, 10.0),
    cluster_frac: float = 0.0,
    cluster_side: int = 64,
    dtype=np.complex64,
    device=None,
    out=None,
) -> DeviceSparseImage:
    """The same workload built in HBM by the library's generator
    (``sfft2d_generate``, csrc/generate.cuh): positions, phases and magnitudes
    are drawn on the host exactly as ``sparse_image`` draws them (same seed ->
    same coefficients), the inverse DFT runs through the library's own FFT, and
    the noise is Philox4x32-10 normals keyed by a 63-bit seed drawn next from
    the same stream.  Noise power uses Parseval, ``mean|x_clean|^2 =
    sum|c|^2 / n^4`` (the host generator's ``np.mean(np.abs(x)**2)`` up to
    roundoff).  ``out``: optional preallocated (n, n) device tensor."""
    from . import _native
    torch = _native._torch()
    _check_side_k(n, k)
    rng = np.random.default_rng(seed)
    rows, cols, coeffs = _draw_spectrum(rng, n, k, magnitude, mag_range, cluster_frac,
                                        cluster_side)
    noise_seed = int(rng.integers(2**63))
    sd = 0.0
    if snr_db is not None:
        power = float(np.sum(np.abs(coeffs) ** 2)) / float(n) ** 4
        sd = float(np.sqrt(power * 10.0 ** (-snr_db / 10.0) / 2.0))
    if np.dtype(dtype) == np.complex64:
        tdt, code = torch.complex64, _native.C64
    elif np.dtype(dtype) == np.complex128:
        tdt, code = torch.complex128, _native.C128
    else:
        raise ValueError(f"unsupported dtype {dtype!r}")
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                       (device.index if isinstance(device, torch.device) else int(device)))
    if out is None:
        out = torch.empty((n, n), dtype=tdt, device=dev)
    elif out.shape != (n, n) or out.dtype != tdt or out.device != dev or not out.is_contiguous():
        raise ValueError("out must be a contiguous (n, n) tensor of the requested dtype on the device")
    ctx = _native.context(dev.index)
    from .tuner import TunerConfig
    tc = TunerConfig()   # the transforms' default tables (any table of side n holds the twiddles)
    ctx.ensure_tables(n, tc.window_delta_pass, tc.window_delta_stop)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    cf = np.ascontiguousarray(coeffs, dtype=np.complex128)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        ctx.check(ctx.lib.sfft2d_generate(ctx.handle, n, int(k), r.ctypes.data, c.ctypes.data,
                                          cf.ctypes.data, sd, noise_seed, code, out.data_ptr(), st))
    return DeviceSparseImage(n, k, seed, out, rows, cols, coeffs, sd, noise_seed)


def planted_image(n: int, k: int, seed: int) -> SparseImage:
    """Noiseless unit-magnitude complex128 image (config c1's workload shape)."""
    return sparse_image(n, k, seed, snr_db=None, dtype=np.complex128)


def error_metric(approx: dict, exact: dict, k: int) -> float:
    """Average L1 spectral error (1/k) * sum |approx - exact| over the union of
    supports, absent entries reading as zero (``signals.py:68-85``)."""
    keys = set(approx) | set(exact)
    total = sum(abs(approx.get(key, 0.0) - exact.get(key, 0.0)) for key in keys)
    if k <= 0:
        return 0.0 if total == 0.0 else float("inf")
    return float(total) / k


def image_digest(x: np.ndarray) -> str:
    """sha256 of the raw bytes; golden fixtures pin regenerated inputs with it."""
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


# SF2D exchange format (signals.py:86-115 of the reference): a 20-byte header
# (magic b"SF2D", n: uint32, k: uint32, seed: uint64, little endian) followed by
# the n*n row-major samples as little-endian float64 (re, im) pairs.  The
# ground truth is not stored.
_SF2D_MAGIC = b"SF2D"
_SF2D_HEADER = struct.Struct("<4sIIQ")


def save_signal(sig: SparseImage, path) -> None:
    """Write ``sig.x`` (any complex dtype, stored as float64 pairs) with its
    (n, k, seed) header."""
    x = np.ascontiguousarray(sig.x, dtype=np.complex128)
    if x.shape != (sig.n, sig.n):
        raise ValueError(f"signal shape {x.shape} does not match n={sig.n}")
    with open(path, "wb") as fh:
        fh.write(_SF2D_HEADER.pack(_SF2D_MAGIC, sig.n, sig.k, sig.seed))
        fh.write(x.view("<f8").tobytes())


def load_signal(path) -> SparseImage:
    """Read an SF2D file; the truth arrays are empty (not stored)."""
    with open(path, "rb") as fh:
        head = fh.read(_SF2D_HEADER.size)
        if len(head) != _SF2D_HEADER.size:
            raise ValueError("truncated SF2D header")
        magic, n, k, seed = _SF2D_HEADER.unpack(head)
        if magic != _SF2D_MAGIC:
            raise ValueError(f"bad magic {magic!r}")
        raw = np.frombuffer(fh.read(), dtype="<f8")
    if raw.size != 2 * n * n:
        raise ValueError(f"payload holds {raw.size} floats, expected {2 * n * n}")
    x = raw.view(np.complex128).reshape(n, n).copy()
    empty = np.empty(0, dtype=np.int64)
    return SparseImage(int(n), int(k), int(seed), x, empty, empty, np.empty(0, np.complex128))
