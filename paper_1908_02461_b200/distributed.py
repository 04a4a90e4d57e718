"""Multi-GPU paths: one process per GPU, torch.distributed
(NCCL) for the plumbing.

* **Loop split** (Algorithm 1, `sfft2d`): the L location loops are independent
  (engine.py:270-273).  Rank r runs loops l = r, r + world, ... through the
  C-ABI location phase (`sfft2d_sfft_votes`), which yields a per-coordinate
  count of the loops that voted it (per-loop dedup, engine.py:144).  One
  all-reduce (sum) of that uint8 histogram is the only collective; every rank
  then thresholds and estimates (`sfft2d_sfft_from_votes`) and returns the same
  dict as single-GPU `sfft2d`.
* **Batch sharding** (config c4): independent images, one shard per rank, no
  data-path collective; `atsfft2d_sharded` gathers the per-image results (small
  Python objects) so every rank ends with the full list in input order.

ATSFFT tuner passes are strictly sequential (tuner.py:182-207) and do not
shard; a single large ATSFFT runs on one GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._tensors import as_device_image
from .batch import atsfft2d_batch
from .engine import ConfigurationError, SfftConfig, _fetch, _stream, to_dict
from .hashing import draw_permutation

__all__ = ["loop_shard", "batch_shard", "merge_votes", "sfft2d_loopsplit", "atsfft2d_sharded",
           "vote_bytes"]


def _dist():
    import torch.distributed as dist
    return dist


def loop_shard(loops: int, rank: int, world: int) -> list:
    """Location loops owned by `rank` (round robin)."""
    return [l for l in range(loops) if l % world == rank]


def batch_shard(n_items: int, rank: int, world: int) -> list:
    """Contiguous block of item indices owned by `rank`."""
    per = (n_items + world - 1) // world
    return list(range(rank * per, min(n_items, (rank + 1) * per)))


def vote_bytes(n: int) -> int:
    """Size of the per-coordinate uint8 vote histogram (padded to 32 keys)."""
    return ((n * n + 31) // 32) * 32


def merge_votes(counts, group=None):
    """Sum the ranks' per-coordinate loop counts in place (the one collective).
    Loops per coordinate <= L <= 255, so uint8 cannot overflow."""
    dist = _dist()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def sfft2d_loopsplit(x, cfg: SfftConfig, rng, *, group=None, precision: str = "fp64",
                     device=None) -> dict:
    """`sfft2d` with the location loops split across the ranks of `group`
    (every rank passes the same x, cfg and rng and gets the same result)."""
    torch = _native._torch()
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    img = as_device_image(x, device)
    if img.n != cfg.n:
        raise ConfigurationError(f"config built for n={cfg.n}, signal has n={img.n}")
    prec = _native.precision_code(precision)
    gen = np.random.default_rng(rng)
    loop_rngs = [np.random.default_rng(int(gen.integers(2**63))) for _ in range(2 * cfg.loops)]
    perms = [draw_permutation(cfg.n, g) for g in loop_rngs]
    mine = loop_shard(cfg.loops, rank, world)
    ctx = _native.context(img.device)
    ctx.ensure_tables(cfg.n, cfg.window_delta_pass, cfg.window_delta_stop)
    ccfg = _native.SfftCfg(cfg.n, cfg.k, cfg.loops, cfg.d_factor, cfg.vote_threshold, cfg.b_bins,
                           cfg.window_delta_pass, cfg.window_delta_stop, cfg.gain_floor,
                           cfg.prune_rel)
    counts = torch.zeros(vote_bytes(cfg.n), dtype=torch.uint8, device=img.tensor.device)
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)
        if mine:
            ctx.check(ctx.lib.sfft2d_sfft_votes(
                ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, ctypes.byref(ccfg),
                _native.perm_array([perms[l] for l in mine]), len(mine), prec, st,
                counts.data_ptr()))
        merge_votes(counts, group)
        res = _native.ResultC()
        ctx.check(ctx.lib.sfft2d_sfft_from_votes(
            ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, ctypes.byref(ccfg),
            counts.data_ptr(), _native.perm_array(perms[cfg.loops:]), prec, st,
            ctypes.byref(res)))
        return to_dict(*_fetch(ctx, res, st, prec))


def atsfft2d_sharded(xs, cfg, est_loops: int, rngs, *, group=None, concurrency: int = 4,
                     precision: str = "fp64", device=None):
    """Batch of independent ATSFFTs sharded over ranks (c4); returns the full
    list of (spectrum, TunerState) in input order on every rank."""
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    idx = batch_shard(len(xs), rank, world)
    local = atsfft2d_batch([xs[i] for i in idx], cfg, est_loops, [rngs[i] for i in idx],
                           concurrency=concurrency, precision=precision, device=device)
    if world == 1:
        return local
    gathered = [None] * world
    dist.all_gather_object(gathered, list(zip(idx, local)), group=group)
    out = [None] * len(xs)
    for part in gathered:
        for i, r in part:
            out[i] = r
    return out
