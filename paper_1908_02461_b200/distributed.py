"""Multi-GPU paths: one process per GPU, torch.distributed
(NCCL) for the plumbing.

* **Loop split** (Algorithm 1, `sfft2d`): the L location loops are independent
  (engine.py:270-273).  Rank r runs loops l = r, r + world, ... through the
  C-ABI location phase (`sfft2d_sfft_votes`), which yields a per-coordinate
  count of the loops that voted it (per-loop dedup, engine.py:144).  One
  all-reduce (sum) of that uint8 histogram merges the votes; every rank
  thresholds it, rank r estimates ITS estimation loops
  (`sfft2d_estimate_loops`), one zero-padded sum all-reduce merges the [L, m]
  estimates and every rank takes the median / top-k / prune
  (`sfft2d_median_select`): the same dict as single-GPU `sfft2d`.
* **Batch sharding** (config c4): independent images, one shard per rank, no
  data-path collective; `atsfft2d_sharded` gathers the per-image results (small
  Python objects) so every rank ends with the full list in input order.

* **Estimation-loop split** (Algorithm 2, `atsfft2d`; the estimation loops
  dominate large configs such as c5, where b_estimate = 8192 and each loop is
  a full hash pass + 8192^2 FFT): the tuner passes are strictly sequential
  (tuner.py:182-207), so every rank runs the same detection (same generator,
  same trajectory), then rank r estimates loops l = r, r + world, ...
  (`sfft2d_estimate_loops`), the per-loop estimates [L, m] are merged with one
  zero-padded sum all-reduce, and every rank takes the median / top-k / prune
  (`sfft2d_median_select`) — the same dict as single-GPU `atsfft2d`.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from ._tensors import as_device_image
from .batch import atsfft2d_batch
from .engine import ConfigurationError, SfftConfig, _fetch, _stream, sfft_perms, to_dict
from .hashing import draw_permutation

__all__ = ["loop_shard", "batch_shard", "merge_votes", "sfft2d_loopsplit", "atsfft2d_sharded",
           "vote_bytes", "merge_estimates", "atsfft2d_loopsplit", "gather_shards", "agree"]


def _dist():
    import torch.distributed as dist
    return dist


def _group_info(group):
    dist = _dist()
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def _all_reduce(t, op, group=None):
    """all_reduce that also works for device tensors on a gloo group (staged
    through host memory; NCCL reduces in place on the device)."""
    dist = _dist()
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


# error classes carried by agree(): a rank-local failure before or between
# collectives must not leave the other ranks blocked in the next all_reduce
_ERR_NONE, _ERR_VALUE, _ERR_CONFIG, _ERR_OTHER = 0, 1, 2, 3


def agree(fn, group=None):
    """Run the rank-local step fn() and agree on its outcome: if any rank
    raised, EVERY rank raises (the same exception class where possible) after
    one small all-reduce, instead of the healthy ranks waiting forever in the
    next collective.  Returns fn()'s value."""
    rank, world = _group_info(group)
    err, out = None, None
    try:
        out = fn()
    except Exception as e:  # noqa: BLE001 - re-raised below on every rank
        err = e
    if world == 1:
        if err is not None:
            raise err
        return out
    torch = _native._torch()
    code = _ERR_NONE if err is None else (
        _ERR_CONFIG if isinstance(err, ConfigurationError) else
        _ERR_VALUE if isinstance(err, ValueError) else _ERR_OTHER)
    dist = _dist()
    on_dev = dist.get_backend(group) == "nccl"
    flag = torch.tensor([code], dtype=torch.int32,
                        device=torch.device("cuda", torch.cuda.current_device()) if on_dev else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    worst = int(flag.item())
    if worst == _ERR_NONE:
        return out
    if err is not None:
        raise err
    msg = f"another rank failed during the split transform (error class {worst})"
    if worst == _ERR_CONFIG:
        raise ConfigurationError(msg)
    if worst == _ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


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
        _all_reduce(counts, dist.ReduceOp.SUM, group)
    return counts


def sfft2d_loopsplit(x, cfg: SfftConfig, rng, *, group=None, precision: str = "fp64",
                     device=None) -> dict:
    """`sfft2d` with the location loops split across the ranks of `group`
    (every rank passes the same x, cfg and rng and gets the same result)."""
    torch = _native._torch()
    rank, world = _group_info(group)
    img = as_device_image(x, device)
    if img.n != cfg.n:
        raise ConfigurationError(f"config built for n={cfg.n}, signal has n={img.n}")
    prec = _native.precision_code(precision)
    perms = sfft_perms(rng, cfg.n, cfg.loops)   # engine.py:266-280, derived natively
    mine = loop_shard(cfg.loops, rank, world)
    ctx = _native.context(img.device)
    ctx.ensure_tables(cfg.n, cfg.window_delta_pass, cfg.window_delta_stop)
    ccfg = _native.SfftCfg(cfg.n, cfg.k, cfg.loops, cfg.d_factor, cfg.vote_threshold, cfg.b_bins,
                           cfg.window_delta_pass, cfg.window_delta_stop, cfg.gain_floor,
                           cfg.prune_rel)
    counts = torch.zeros(vote_bytes(cfg.n), dtype=torch.uint8, device=img.tensor.device)
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)

        def location():
            if mine:   # the native location phase checks for NaN/Inf first
                ctx.check(ctx.lib.sfft2d_sfft_votes(
                    ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, ctypes.byref(ccfg),
                    _native.perm_array([perms[l] for l in mine]), len(mine), prec, st,
                    counts.data_ptr()))
            elif not bool(torch.isfinite(torch.view_as_real(img.tensor)).all()):
                # a rank without location loops still validates its input
                # (as_complex_matrix, corefft.py:49-50) so every rank agrees
                raise ValueError("matrix contains NaN or Inf")

        agree(location, group)
        merge_votes(counts, group)
        # estimation loops split too: candidates = coordinates voted by at
        # least vote_threshold loops (ascending, engine.py:148-160); rank r
        # estimates loops l = r, r + world, ...; one sum all-reduce merges the
        # [L, m] table; every rank takes the median / top-k / prune
        keys = torch.nonzero(counts[: cfg.n * cfg.n] >= cfg.vote_threshold).flatten().to(torch.int32)
        m = int(keys.numel())
        if m == 0:
            return {}
        est = perms[cfg.loops:]
        cdt = torch.complex128 if prec == _native.FP64 else torch.complex64
        vals = torch.zeros((cfg.loops, m), dtype=cdt, device=counts.device)
        usable = torch.zeros((cfg.loops, m), dtype=torch.uint8, device=counts.device)

        def estimation():
            if not mine:
                return
            lv = torch.empty((len(mine), m), dtype=cdt, device=counts.device)
            lu = torch.empty((len(mine), m), dtype=torch.uint8, device=counts.device)
            ctx.check(ctx.lib.sfft2d_estimate_loops(
                ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, cfg.n, cfg.b_bins,
                cfg.window_delta_pass, cfg.window_delta_stop, cfg.gain_floor, keys.data_ptr(), m,
                _native.perm_array([est[l] for l in mine]), len(mine), prec, st, lv.data_ptr(),
                lu.data_ptr()))
            idx = torch.as_tensor(mine, device=counts.device)
            vals.index_copy_(0, idx, lv)
            usable.index_copy_(0, idx, lu)

        agree(estimation, group)
        merge_estimates(vals, usable, group)
        res = _native.ResultC()
        ctx.check(ctx.lib.sfft2d_median_select(
            ctx.handle, cfg.n, keys.data_ptr(), m, vals.data_ptr(), usable.data_ptr(), cfg.loops,
            cfg.k, cfg.prune_rel, prec, st, ctypes.byref(res)))
        return to_dict(*_fetch(ctx, res, st, prec))


def atsfft2d_sharded(xs, cfg, est_loops: int, rngs, *, group=None, concurrency: int = 4,
                     precision: str = "fp64", device=None):
    """Batch of independent ATSFFTs sharded over ranks (c4); returns the full
    list of (spectrum, TunerState) in input order on every rank."""
    rank, world = _group_info(group)
    if len(xs) != len(rngs):
        raise ValueError("need one rng per image")
    idx = batch_shard(len(xs), rank, world)
    local = agree(lambda: atsfft2d_batch([xs[i] for i in idx], cfg, est_loops,
                                         [rngs[i] for i in idx], concurrency=concurrency,
                                         precision=precision, device=device), group)
    return gather_shards(idx, local, len(xs), group)


def gather_shards(idx, local, n_items: int, group=None) -> list:
    """Every rank's (item index, result) pairs gathered into the full list in
    input order, on every rank (results are small Python objects)."""
    rank, world = _group_info(group)
    if world == 1:
        out = [None] * n_items
        for i, r in zip(idx, local):
            out[i] = r
        return out
    gathered = [None] * world
    _dist().all_gather_object(gathered, list(zip(idx, local)), group=group)
    out = [None] * n_items
    for part in gathered:
        for i, r in part:
            out[i] = r
    return out


def merge_estimates(vals, usable, group=None):
    """Zero-padded sum all-reduce of per-loop estimates: every rank filled only
    the rows [l] of the loops it owns (others zero), so the sum is the full
    [L, m] table (complex values as their real view) and usable flags."""
    dist = _dist()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        torch = _native._torch()
        re = torch.view_as_real(vals) if vals.is_complex() else vals
        _all_reduce(re, dist.ReduceOp.SUM, group)
        _all_reduce(usable, dist.ReduceOp.SUM, group)
    return vals, usable


def atsfft2d_loopsplit(x, cfg, est_loops: int, rng, *, group=None, precision: str = "fp64",
                       device=None):
    """`atsfft2d` with the estimation loops split across the ranks of `group`
    (every rank passes the same x, cfg, est_loops and seed, and gets the same
    (dict, TunerState) as single-GPU `atsfft2d`, tuner.py:244-282).  A
    Generator passed as `rng` advances exactly as under the reference."""
    from .tuner import _run_ats
    torch = _native._torch()
    rank, world = _group_info(group)
    gen = rng if isinstance(rng, np.random.Generator) else np.random.default_rng(rng)
    img = as_device_image(x, device)
    n = img.n
    # detection with the votes left on the device (the reference's
    # detect_sparsity, tuner.py:142-241); candidates = tally >= threshold,
    # ascending keys i*n + j (engine.py:148-160 order)
    state, (vkeys, vtal) = agree(lambda: _run_ats(img.tensor, cfg, 0, gen, precision, img.device,
                                                  False, on_device=True), group)
    if state.detected_k == 0 or vkeys.numel() == 0:
        return {}, state
    thr = (max(state.vote_passes, 1) + 1) // 2
    keys = vkeys[vtal >= thr].contiguous()
    if keys.numel() == 0:
        return {}, state
    ecfg = SfftConfig(n=n, k=state.detected_k, loops=max(int(est_loops), 1),
                      b_bins=state.b_estimate, window_delta_pass=cfg.window_delta_pass,
                      window_delta_stop=cfg.window_delta_stop, gain_floor=cfg.gain_floor,
                      prune_rel=cfg.prune_rel)          # ConfigurationError as the reference
    perms = [draw_permutation(n, gen) for _ in range(ecfg.loops)]
    prec = _native.precision_code(precision)
    L, m = ecfg.loops, int(keys.numel())
    if ecfg.b_bins == n:
        # all-pass window: every loop returns x_hat[i, j] itself (gain 1, the
        # phase twists cancel; Lemma 1), so one loop on every rank is the
        # median of all of them up to roundoff — nothing to split
        L, perms = 1, perms[:1]
    dev = img.tensor.device
    cdt = torch.complex128 if prec == _native.FP64 else torch.complex64
    vals = torch.zeros((L, m), dtype=cdt, device=dev)
    usable = torch.zeros((L, m), dtype=torch.uint8, device=dev)
    mine = [0] if L == 1 else loop_shard(L, rank, world)
    ctx = _native.context(img.device)
    ctx.ensure_tables(n, cfg.window_delta_pass, cfg.window_delta_stop)
    with torch.cuda.device(img.device):
        st = _stream(torch, img.device)

        def estimation():
            if not mine:
                return
            lv = torch.empty((len(mine), m), dtype=cdt, device=dev)
            lu = torch.empty((len(mine), m), dtype=torch.uint8, device=dev)
            ctx.check(ctx.lib.sfft2d_estimate_loops(
                ctx.handle, img.tensor.data_ptr(), img.dtype_code, 0, n, ecfg.b_bins,
                ecfg.window_delta_pass, ecfg.window_delta_stop, ecfg.gain_floor, keys.data_ptr(), m,
                _native.perm_array([perms[l] for l in mine]), len(mine), prec, st,
                lv.data_ptr(), lu.data_ptr()))
            idx = torch.as_tensor(mine, device=dev)
            vals.index_copy_(0, idx, lv)
            usable.index_copy_(0, idx, lu)

        if L > 1:
            agree(estimation, group)
        else:
            estimation()
        if L > 1:
            merge_estimates(vals, usable, group)
        res = _native.ResultC()
        ctx.check(ctx.lib.sfft2d_median_select(
            ctx.handle, n, keys.data_ptr(), m, vals.data_ptr(), usable.data_ptr(), L,
            int(state.detected_k), ecfg.prune_rel, prec, st, ctypes.byref(res)))
        return to_dict(*_fetch(ctx, res, st, prec)), state
