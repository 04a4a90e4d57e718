"""CPU restatement of the device workload generator (test infrastructure only).

Restates ``paper_1908_02461_b200/csrc/generate.cuh`` (``sfft2d_generate``):
Philox4x32-10 keyed by the 64-bit noise seed with counter = flat element index,
two 53-bit uniforms per element, Box-Muller in double, and the clean image
``ifft2(S)`` (``corefft.py:112-118`` convention) from numpy's float64 FFT.  The
reference has no device generator (its generator is host-side,
``/root/reference/pkg/src/sfft2d/signals.py:42-65``); this file pins the
device stream so the GPU tests can compare the device image with it.

Philox4x32-10 is the published counter-based generator of Salmon et al.
(SC'11, "Parallel random numbers: as easy as 1, 2, 3"); the known-answer
vectors in tests/test_generator.py are that paper's Random123 KAT values.
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(ctr, key):
    """Vectorised Philox4x32-10: ctr uint32[..., 4], key (k0, k1) -> uint32[..., 4]."""
    c = [np.asarray(ctr[..., i], dtype=np.uint64) for i in range(4)]
    k0, k1 = int(key[0]) & 0xFFFFFFFF, int(key[1]) & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return np.stack([v.astype(np.uint32) for v in c], axis=-1)


def noise(total: int, seed: int):
    """(n1, n2) standard normals for flat elements 0..total-1 (generate.cuh k_gen_finish)."""
    e = np.arange(total, dtype=np.uint64)
    ctr = np.zeros((total, 4), dtype=np.uint64)
    ctr[:, 0] = e & MASK
    ctr[:, 1] = e >> np.uint64(32)
    r = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)).astype(np.uint64)
    scale = 1.0 / 9007199254740992.0
    u1 = 1.0 - (((r[:, 0] >> np.uint64(5)) << np.uint64(26)) | (r[:, 1] >> np.uint64(6))).astype(
        np.float64) * scale
    u2 = (((r[:, 2] >> np.uint64(5)) << np.uint64(26)) | (r[:, 3] >> np.uint64(6))).astype(
        np.float64) * scale
    rad = np.sqrt(-2.0 * np.log(u1))
    return rad * np.cos(2.0 * np.pi * u2), rad * np.sin(2.0 * np.pi * u2)


def device_image(n, rows, cols, coeffs, noise_sd, noise_seed, dtype=np.complex64):
    """The image sfft2d_generate writes, computed on the host in float64."""
    spec = np.zeros((n, n), dtype=np.complex128)
    spec[np.asarray(rows), np.asarray(cols)] = coeffs
    x = np.fft.ifft2(spec)
    if noise_sd > 0:
        n1, n2 = noise(n * n, int(noise_seed))
        x = x + noise_sd * (n1 + 1j * n2).reshape(n, n)
    return x.astype(dtype)
