"""PyTorch custom operators over the C ABI.

Importing this module registers ``torch.ops.sfft2d_b200.*`` — each a thin call
into ``libsfft2d_b200.so`` on CUDA tensors, with a fake (meta) kernel so the
ops trace under ``torch.compile`` / ``make_fx`` (data-dependent output sizes
are dynamic).  Permutations are int64 tensors ``[L, 6]`` = (σ1, σ2, τ1, τ2,
σ1⁻¹, σ2⁻¹) as in ``hashing.PermutationParams``; ``fp64`` selects the
arithmetic (the reference's float64, or the fp32 fast path).

    binned_spectrum(x, perms, b, delta_pass, delta_stop, fp64) -> [L, b, b]   hashing.py:308-337
    bucket_fft2d(grids, n_table, fp64) -> [count, b, b]                       corefft.py:101-109
    top_bins(grids, num, fp64) -> int32 [nseg, num]                           engine.py:122-127
    local_maxima(grid, mag_floor, fp64) -> int64 [m, 2]                       tuner.py:97-118
    sfft(x, seed, k, loops, ..., fp64) -> (int64 [m, 2], complex [m])         engine.py:256-284
    atsfft(x, seed, est_loops, b0, ..., fp64) -> (int64 [m, 2], complex [m])  tuner.py:244-282
"""

from __future__ import annotations

import ctypes
from types import SimpleNamespace

import torch

from . import _native
from .engine import _stream, sfft2d_arrays, SfftConfig
from .tuner import TunerConfig, atsfft2d_arrays, count_local_maxima

__all__ = ["binned_spectrum", "bucket_fft2d", "top_bins", "local_maxima", "sfft", "atsfft"]

_NS = "sfft2d_b200"


def _cdtype(fp64: bool):
    return torch.complex128 if fp64 else torch.complex64


def _prec(fp64: bool) -> int:
    return _native.FP64 if fp64 else _native.FP32


def _perm_objs(perms: torch.Tensor):
    rows = perms.detach().to("cpu", torch.int64).reshape(-1, 6).tolist()
    return [SimpleNamespace(sigma1=r[0], sigma2=r[1], tau1=r[2], tau2=r[3], sigma1_inv=r[4],
                            sigma2_inv=r[5]) for r in rows]


def _cuda_ctx(t: torch.Tensor):
    if t.device.type != "cuda":
        raise ValueError("sfft2d_b200 ops take CUDA tensors")
    return _native.context(t.device.index)


# ------------------------------------------------------------- binned spectrum
@torch.library.custom_op(f"{_NS}::binned_spectrum", mutates_args=())
def binned_spectrum(x: torch.Tensor, perms: torch.Tensor, b: int, delta_pass: float,
                    delta_stop: float, fp64: bool) -> torch.Tensor:
    ctx = _cuda_ctx(x)
    n = int(x.shape[-1])
    if x.dim() != 2 or x.shape[0] != n:
        raise ValueError("x must be a square N x N complex tensor")
    xc = x.contiguous()
    code = _native.C128 if xc.dtype == torch.complex128 else _native.C64
    if xc.dtype not in (torch.complex64, torch.complex128):
        xc, code = xc.to(torch.complex128), _native.C128
    plist = _perm_objs(perms)
    ctx.ensure_tables(n, delta_pass, delta_stop)
    out = torch.empty((len(plist), b, b), dtype=_cdtype(fp64), device=x.device)
    with torch.cuda.device(x.device):
        st = _stream(torch, x.device.index)
        ctx.check(ctx.lib.sfft2d_binned_spectrum(ctx.handle, xc.data_ptr(), code, n, b,
                                                 _native.perm_array(plist), len(plist),
                                                 float(delta_pass), float(delta_stop),
                                                 _prec(fp64), out.data_ptr(), st))
    return out


@binned_spectrum.register_fake
def _(x, perms, b, delta_pass, delta_stop, fp64):
    return x.new_empty((perms.shape[0], b, b), dtype=_cdtype(fp64))


# ------------------------------------------------------------- bucket FFT
@torch.library.custom_op(f"{_NS}::bucket_fft2d", mutates_args=())
def bucket_fft2d(grids: torch.Tensor, n_table: int, fp64: bool) -> torch.Tensor:
    ctx = _cuda_ctx(grids)
    b = int(grids.shape[-1])
    out = grids.reshape(-1, b, b).to(_cdtype(fp64)).contiguous().clone()
    ctx.ensure_tables(int(n_table), 1e-3, 1e-8)
    with torch.cuda.device(grids.device):
        st = _stream(torch, grids.device.index)
        ctx.check(ctx.lib.sfft2d_fft2d(ctx.handle, out.data_ptr(), b, out.shape[0], int(n_table),
                                       _prec(fp64), st))
    return out


@bucket_fft2d.register_fake
def _(grids, n_table, fp64):
    b = grids.shape[-1]
    return grids.new_empty((grids.numel() // (b * b), b, b), dtype=_cdtype(fp64))


# ------------------------------------------------------------- top bins
@torch.library.custom_op(f"{_NS}::top_bins", mutates_args=())
def top_bins(grids: torch.Tensor, num: int, fp64: bool) -> torch.Tensor:
    ctx = _cuda_ctx(grids)
    b = int(grids.shape[-1])
    g = grids.reshape(-1, b, b).to(_cdtype(fp64)).contiguous()
    out = torch.empty((g.shape[0], num), dtype=torch.int32, device=grids.device)
    with torch.cuda.device(grids.device):
        st = _stream(torch, grids.device.index)
        ctx.check(ctx.lib.sfft2d_top_bins(ctx.handle, g.data_ptr(), b, g.shape[0], int(num),
                                          _prec(fp64), out.data_ptr(), st))
    return out


@top_bins.register_fake
def _(grids, num, fp64):
    b = grids.shape[-1]
    return grids.new_empty((grids.numel() // (b * b), num), dtype=torch.int32)


# ------------------------------------------------------------- local maxima
@torch.library.custom_op(f"{_NS}::local_maxima", mutates_args=())
def local_maxima(grid: torch.Tensor, mag_floor: float, fp64: bool) -> torch.Tensor:
    _cuda_ctx(grid)
    _, coords = count_local_maxima(grid, mag_floor, precision="fp64" if fp64 else "fp32")
    return torch.from_numpy(coords).to(grid.device)


@local_maxima.register_fake
def _(grid, mag_floor, fp64):
    m = torch.library.get_ctx().new_dynamic_size()
    return grid.new_empty((m, 2), dtype=torch.int64)


# ------------------------------------------------------------- whole transforms
@torch.library.custom_op(f"{_NS}::sfft", mutates_args=())
def sfft(x: torch.Tensor, seed: int, k: int, loops: int, d_factor: int, vote_threshold: int,
         b_bins: int, delta_pass: float, delta_stop: float, gain_floor: float, prune_rel: float,
         fp64: bool) -> tuple[torch.Tensor, torch.Tensor]:
    _cuda_ctx(x)
    cfg = SfftConfig(n=int(x.shape[-1]), k=k, loops=loops, d_factor=d_factor,
                     vote_threshold=vote_threshold if vote_threshold > 0 else None,
                     b_bins=b_bins if b_bins > 0 else None, window_delta_pass=delta_pass,
                     window_delta_stop=delta_stop, gain_floor=gain_floor, prune_rel=prune_rel)
    ij, vals = sfft2d_arrays(x, cfg, seed, precision="fp64" if fp64 else "fp32")
    return torch.from_numpy(ij).to(x.device), torch.from_numpy(vals).to(x.device)


@sfft.register_fake
def _(x, seed, k, loops, d_factor, vote_threshold, b_bins, delta_pass, delta_stop, gain_floor,
      prune_rel, fp64):
    m = torch.library.get_ctx().new_dynamic_size()
    return x.new_empty((m, 2), dtype=torch.int64), x.new_empty((m,), dtype=_cdtype(fp64))


@torch.library.custom_op(f"{_NS}::atsfft", mutates_args=())
def atsfft(x: torch.Tensor, seed: int, est_loops: int, b0: int, eps1: float, eps2: float,
           delta1: float, delta2: float, max_tuning_iters: int, mag_floor: float,
           delta_pass: float, delta_stop: float, gain_floor: float, prune_rel: float,
           fp64: bool) -> tuple[torch.Tensor, torch.Tensor]:
    _cuda_ctx(x)
    cfg = TunerConfig(b0=b0, eps1=eps1, eps2=eps2, delta1=delta1, delta2=delta2,
                      max_tuning_iters=None if max_tuning_iters < 0 else max_tuning_iters,
                      mag_floor=mag_floor, window_delta_pass=delta_pass,
                      window_delta_stop=delta_stop, gain_floor=gain_floor, prune_rel=prune_rel)
    (ij, vals), _ = atsfft2d_arrays(x, cfg, est_loops, seed, precision="fp64" if fp64 else "fp32")
    return torch.from_numpy(ij).to(x.device), torch.from_numpy(vals).to(x.device)


@atsfft.register_fake
def _(x, seed, est_loops, b0, eps1, eps2, delta1, delta2, max_tuning_iters, mag_floor, delta_pass,
      delta_stop, gain_floor, prune_rel, fp64):
    m = torch.library.get_ctx().new_dynamic_size()
    return x.new_empty((m, 2), dtype=torch.int64), x.new_empty((m,), dtype=_cdtype(fp64))


def perms_tensor(perms) -> torch.Tensor:
    """[L, 6] int64 tensor from ``PermutationParams`` objects."""
    return torch.tensor([[p.sigma1, p.sigma2, p.tau1, p.tau2, p.sigma1_inv, p.sigma2_inv]
                         for p in perms], dtype=torch.int64)


__all__.append("perms_tensor")
_ = ctypes  # the ABI calls above pass plain pointers
