"""The reference's lower-level Algorithm 1 building blocks (engine.py:130-220):
``seek_location_once`` / ``estimate_once`` on the GPU against the oracle, and
the host-side ``vote_and_select`` / ``median_combine`` against the oracle's
restatement, plus the composed pipeline equal to ``sfft2d``."""

import numpy as np
import pytest
import torch

import paper_1908_02461_b200 as P
from oracle import sfft_oracle as O

gpu = pytest.mark.gpu


def test_vote_and_select_matches_oracle():
    rng = np.random.default_rng(4)
    n = 64
    cfg = P.SfftConfig(n=n, k=3, loops=5)
    sets = [np.stack(np.unravel_index(np.unique(rng.integers(0, n * n, 40)), (n, n)), axis=1)
            for _ in range(cfg.loops)]
    got = P.vote_and_select(sets, cfg)
    want = O.vote([s[:, 0] * n + s[:, 1] for s in sets], cfg.vote_threshold)
    np.testing.assert_array_equal(got[:, 0] * n + got[:, 1], want)
    with pytest.raises(ValueError):
        P.vote_and_select(sets[:-1], cfg)


def test_median_combine_semantics():
    ests = [{(0, 1): 1 + 1j, (2, 3): 5.0}, {(0, 1): 3 - 1j}, {(0, 1): 2 + 4j, (4, 4): -1j}]
    out = P.median_combine(ests)
    assert list(out) == [(0, 1), (2, 3), (4, 4)]
    assert out[(0, 1)] == complex(2, 1) and out[(2, 3)] == 5.0 and out[(4, 4)] == -1j
    # explicit coordinates: order kept, coordinates without estimates dropped
    out2 = P.median_combine(ests[:2], coords=[(2, 3), (9, 9), (0, 1)])
    assert list(out2) == [(2, 3), (0, 1)] and out2[(0, 1)] == complex(2, 0)


@gpu
def test_seek_location_once_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sig = P.planted_image(256, 6, 3)
    cfg = P.SfftConfig(n=256, k=6)
    win = P.build_flat_window(256, cfg.b_bins, cfg.window_delta_stop,
                              delta_pass=cfg.window_delta_pass)
    p, cand = P.seek_location_once(sig.x, cfg, win, 11)
    gen = np.random.default_rng(11)
    q = O.draw_perm(256, gen)
    assert (p.sigma1, p.sigma2, p.tau1, p.tau2) == (q.s1, q.s2, q.t1, q.t2)
    ow = O.window(256, cfg.b_bins, cfg.window_delta_stop, cfg.window_delta_pass)
    keys = O.location_loop(O.as_c128(sig.x), O.sfft_params(256, 6), ow, q)
    np.testing.assert_array_equal(cand[:, 0] * 256 + cand[:, 1], keys)


@gpu
def test_estimate_once_matches_oracle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    img = P.sparse_image(256, 8, 5, snr_db=25.0, dtype=np.complex128)
    cfg = P.SfftConfig(n=256, k=8)
    win = P.build_flat_window(256, cfg.b_bins, cfg.window_delta_stop,
                              delta_pass=cfg.window_delta_pass)
    p = P.draw_permutation(256, np.random.default_rng(2))
    coords = np.concatenate([np.stack([img.rows, img.cols], axis=1),
                             np.random.default_rng(0).integers(0, 256, (40, 2))])
    got = P.estimate_once(img.x, coords, p, win, cfg)
    q = O.make_perm(256, p.sigma1, p.sigma2, p.tau1, p.tau2)
    ow = O.window(256, cfg.b_bins, cfg.window_delta_stop, cfg.window_delta_pass)
    vals, ok = O.estimate(O.as_c128(img.x), coords, q, ow, cfg.b_bins, cfg.gain_floor)
    want = {(int(i), int(j)): complex(v) for (i, j), v, u in zip(coords, vals, ok) if u}
    assert set(got) == set(want)
    for key, v in want.items():
        assert abs(got[key] - v) <= 1e-10 * max(1.0, abs(v))


@gpu
def test_composed_pipeline_recovers_planted_support():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sig = P.planted_image(256, 6, 3)
    cfg = P.SfftConfig(n=256, k=6)
    win = P.build_flat_window(256, cfg.b_bins, cfg.window_delta_stop,
                              delta_pass=cfg.window_delta_pass)
    gen = np.random.default_rng(7)
    sets = [P.seek_location_once(sig.x, cfg, win, gen)[1] for _ in range(cfg.loops)]
    coords = P.vote_and_select(sets, cfg)
    ests = [P.estimate_once(sig.x, coords, P.draw_permutation(256, gen), win, cfg)
            for _ in range(cfg.loops)]
    med = P.median_combine(ests, coords)
    top = sorted(med, key=lambda k: -abs(med[k]))[:6]
    assert set(top) == set(sig.truth)
    for key in top:
        assert abs(med[key] - sig.truth[key]) < 1e-6


@pytest.mark.gpu
def test_caller_owned_workspace():
    # the caller (torch) owns the device workspace; the
    # library sub-allocates it, reports the size a workload needs, and fails
    # with a status (no allocation of its own) when it is too small
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1908_02461_b200 import _native
    img = P.sparse_image(1024, 30, 3, snr_db=25.0)
    x = torch.from_numpy(img.x).cuda()
    ctx = _native.context()
    ref, rs = P.atsfft2d(x, P.TunerConfig(), 8, 5)
    _, peak = ctx.workspace_size()
    assert peak > 0
    buf = torch.empty(2 * peak, dtype=torch.uint8, device="cuda")
    try:
        ctx.use_workspace(buf)
        got, gs = P.atsfft2d(x, P.TunerConfig(), 8, 5)
        assert got == ref and gs == rs
        assert 0 < ctx.workspace_size()[1] <= buf.numel()
        ctx.use_workspace(torch.empty(1 << 16, dtype=torch.uint8, device="cuda"))
        with pytest.raises(_native.StatusError, match="workspace exhausted"):
            P.atsfft2d(x, P.TunerConfig(), 8, 5)
    finally:
        ctx.use_workspace(None)
    again, _ = P.atsfft2d(x, P.TunerConfig(), 8, 5)
    assert again == ref


def _median_select_gpu(n, keys, vals, usable, k, prune_rel, precision="fp64"):
    """sfft2d_median_select (K7: median, top-k cut with ties to the lowest index,
    prune, ordered output) through the C ABI."""
    import ctypes
    from paper_1908_02461_b200 import _native
    from paper_1908_02461_b200.engine import _fetch, _stream, to_dict
    prec = _native.precision_code(precision)
    cdt = torch.complex128 if precision == "fp64" else torch.complex64
    ctx = _native.context(0)
    kd = torch.from_numpy(keys.astype(np.int32)).cuda()
    vd = torch.from_numpy(vals).to(cdt).cuda().contiguous()
    ud = torch.from_numpy(usable.astype(np.uint8)).cuda().contiguous()
    res = _native.ResultC()
    st = _stream(torch, 0)
    ctx.check(ctx.lib.sfft2d_median_select(ctx.handle, n, kd.data_ptr(), int(keys.size), vd.data_ptr(),
                                           ud.data_ptr(), int(vals.shape[0]), int(k), float(prune_rel),
                                           prec, st, ctypes.byref(res)))
    return to_dict(*_fetch(ctx, res, st, prec))


@gpu
@pytest.mark.parametrize("m,k,prune", [(500, 100, 0.0), (500, 100, 0.4), (3000, 7, 0.0),
                                       (16384, 4000, 0.3), (40000, 9000, 0.0), (300, 1000, 0.5)])
def test_median_select_ties_match_oracle(m, k, prune):
    """Magnitudes drawn from a handful of exact values, so the top-k cut is
    decided by ties almost everywhere (engine.py:245-253: lexsort(-|v|, i, j):
    ties to the lowest coordinate), some loops unusable, some coordinates dead
    in every loop; m <= 16384 runs the one-CTA tail (k_finish_cut_small),
    larger m the multi-launch selection.  Support, values and dict order must
    equal the oracle's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    n, L = 256, 5
    rng = np.random.default_rng(m + k)
    keys = np.sort(rng.choice(n * n, size=m, replace=False))
    coords = np.stack([keys // n, keys % n], axis=1).astype(np.int64)
    mags = rng.choice([1.0, 2.0, 2.0, 3.0, 0.5], size=m)
    phase = rng.choice([1, -1, 1j, -1j], size=m)
    base = mags * phase
    # every loop reports the same value where usable, so the median is exactly
    # `base` and equal magnitudes are equal to the last bit
    vals = np.tile(base, (L, 1)).astype(np.complex128)
    usable = rng.random((L, m)) < 0.7
    usable[:, rng.random(m) < 0.1] = False           # dead coordinates
    vals[~usable] = 0.0
    got = _median_select_gpu(n, keys, vals, usable, k, prune)
    cs, med = O.median_pick(coords, [v for v in vals], [u for u in usable], k, prune)
    want = O.as_dict((cs, med))
    assert list(got) == list(want)
    assert all(got[key] == v for key, v in want.items())
