"""Multi-process (world_size 2) tests of the distributed host logic on CPU
with the gloo backend: loop sharding + the vote-histogram all-reduce of the
loop-split SFFT, and batch sharding + result gathering.  The per-rank compute
is the oracle (no GPU here); the merge/shard code is the product's."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sfft_oracle as O
from paper_1908_02461_b200 import distributed as D
from paper_1908_02461_b200.signals import planted_image, sparse_image


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _loop_counts(x, cfg, seed, loops):
    """Per-coordinate loop-vote counts of the given location loops (oracle)."""
    a = O.as_c128(x)
    gen = np.random.default_rng(seed)
    kids = [np.random.default_rng(int(gen.integers(2**63))) for _ in range(2 * cfg.loops)]
    win = O.cached_window(cfg.n, cfg.b, cfg.dstop, cfg.dpass)
    counts = np.zeros(D.vote_bytes(cfg.n), dtype=np.uint8)
    for l in loops:
        keys = O.location_loop(a, cfg, win, O.draw_perm(cfg.n, kids[l]))
        counts[keys] += 1
    return counts


def _worker_votes(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sig = planted_image(128, 6, 3)
    cfg = O.sfft_params(128, 6, loops=7)
    mine = D.loop_shard(cfg.loops, rank, world)
    counts = torch.from_numpy(_loop_counts(sig.x, cfg, 5, mine))
    D.merge_votes(counts)
    if rank == 0:
        np.save(out_path, counts.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_loopsplit_vote_allreduce_matches_single_process():
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "counts.npy")
        mp.spawn(_worker_votes, args=(2, _free_port(), out), nprocs=2, join=True)
        merged = np.load(out)
    sig = planted_image(128, 6, 3)
    cfg = O.sfft_params(128, 6, loops=7)
    full = _loop_counts(sig.x, cfg, 5, range(cfg.loops))
    np.testing.assert_array_equal(merged, full)
    # thresholding the merged histogram reproduces the single-process vote
    (_, _), trace = O.sfft(sig.x, cfg, 5, return_trace=True)
    voted = np.flatnonzero(merged[: 128 * 128] >= cfg.threshold)
    np.testing.assert_array_equal(voted, trace["keys"])


def _worker_batch(rank, world, port, out_path):
    # the product's shard + gather (D.batch_shard, D.agree, D.gather_shards, the
    # code atsfft2d_sharded runs around its per-rank GPU batch), with the oracle
    # as the per-rank compute
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_items = 5
    idx = D.batch_shard(n_items, rank, world)

    def compute():
        local = []
        for i in idx:
            img = sparse_image(64, 3, 10 + i, snr_db=25.0)
            (cs, vs), st = O.atsfft(img.x, O.TunerParams(), 4, 20 + i)
            local.append((cs.tolist(), [complex(v) for v in vs], st["detected_k"]))
        return local

    out = D.gather_shards(idx, D.agree(compute), n_items)
    if rank == 0:
        torch.save(out, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_batch_shard_gather_matches_sequential():
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "res.pt")
        mp.spawn(_worker_batch, args=(2, _free_port(), out), nprocs=2, join=True)
        got = torch.load(out, weights_only=False)
    for i in range(5):
        img = sparse_image(64, 3, 10 + i, snr_db=25.0)
        (cs, vs), st = O.atsfft(img.x, O.TunerParams(), 4, 20 + i)
        assert got[i] == (cs.tolist(), [complex(v) for v in vs], st["detected_k"])


def _worker_agree(rank, world, port, out_path):
    # a failure on ONE rank before a collective makes every rank raise (no
    # rank left blocked in the next all_reduce); ValueError class preserved
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def step():
        if rank == 1:
            raise ValueError("matrix contains NaN or Inf")
        return 7

    try:
        D.agree(step)
        outcome = "returned"
    except ValueError as e:
        outcome = f"ValueError:{e}"
    ok = D.agree(lambda: 3)
    torch.save((outcome, ok), out_path + f".{rank}")
    dist.barrier()
    dist.destroy_process_group()


def test_agree_raises_on_every_rank():
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "agree")
        mp.spawn(_worker_agree, args=(2, _free_port(), out), nprocs=2, join=True)
        r0, r1 = torch.load(out + ".0"), torch.load(out + ".1")
    assert r0[0].startswith("ValueError:another rank failed") and r0[1] == 3
    assert r1 == ("ValueError:matrix contains NaN or Inf", 3)


def test_shards_partition():
    for world in (1, 2, 3, 8):
        loops = [D.loop_shard(8, r, world) for r in range(world)]
        assert sorted(sum(loops, [])) == list(range(8))
        items = [D.batch_shard(2048, r, world) for r in range(world)]
        assert sum(items, []) == list(range(2048))


@pytest.mark.gpu
def test_loopsplit_single_gpu_equals_sfft2d():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1908_02461_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for n, k, seed in ((256, 10, 1), (1024, 30, 2)):
            img = sparse_image(n, k, seed, snr_db=25.0)
            cfg = P.SfftConfig(n=n, k=k)
            a = P.sfft2d(img.x, cfg, 9)
            b = D.sfft2d_loopsplit(img.x, cfg, 9)
            assert a == b
    finally:
        dist.destroy_process_group()


def _est_case():
    img = sparse_image(128, 5, 41, snr_db=20.0)
    a = O.as_c128(img.x)
    gen = np.random.default_rng(43)
    state, (vc, vt), _ = O.detect(a, O.TunerParams(), gen)
    thr = (max(state["vote_passes"], 1) + 1) // 2
    coords = vc[vt >= thr]
    ecfg = O.sfft_params(128, state["detected_k"], loops=6, b_bins=state["b_estimate"])
    win = O.cached_window(128, ecfg.b, ecfg.dstop, ecfg.dpass)
    perms = [O.draw_perm(128, gen) for _ in range(ecfg.loops)]
    return a, coords, ecfg, win, perms, state


def _worker_est(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, coords, ecfg, win, perms, _ = _est_case()
    vals = torch.zeros((ecfg.loops, len(coords)), dtype=torch.complex128)
    usable = torch.zeros((ecfg.loops, len(coords)), dtype=torch.uint8)
    for l in D.loop_shard(ecfg.loops, rank, world):   # this rank's estimation loops only
        v, o = O.estimate(a, coords, perms[l], win, ecfg.b, ecfg.gain_floor)
        vals[l] = torch.from_numpy(np.asarray(v, dtype=np.complex128))
        usable[l] = torch.from_numpy(np.asarray(o, dtype=np.uint8))
    D.merge_estimates(vals, usable)
    if rank == 0:
        torch.save((vals, usable), out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_estimation_split_merge_matches_single_process():
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "est.pt")
        mp.spawn(_worker_est, args=(2, _free_port(), out), nprocs=2, join=True)
        vals, usable = torch.load(out)
    a, coords, ecfg, win, perms, state = _est_case()
    vl, ol = zip(*[O.estimate(a, coords, p, win, ecfg.b, ecfg.gain_floor) for p in perms])
    np.testing.assert_array_equal(vals.numpy(), np.asarray(vl, dtype=np.complex128))
    np.testing.assert_array_equal(usable.numpy().astype(bool), np.asarray(ol, dtype=bool))
    # the median / top-k / prune over the merged table is the reference's result
    got = O.median_pick(coords, list(vals.numpy()), list(usable.numpy().astype(bool)),
                        state["detected_k"], O.TunerParams().prune_rel)
    ref, _ = O.atsfft(a, O.TunerParams(), 6, 43)
    assert O.as_dict(got) == O.as_dict(ref)


@pytest.mark.gpu
def test_atsfft_estimation_split_single_gpu_equals_atsfft2d():
    # world size 1 through the split entry points (sfft2d_estimate_loops +
    # sfft2d_median_select, NCCL process group): the same support and values as
    # atsfft2d, the reference's result, and the same Generator advance
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1908_02461_b200 as P
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for n, k, seed in ((512, 9, 3), (256, 20, 4), (1024, 50, 7)):
            img = sparse_image(n, k, seed, snr_db=25.0)
            g1, g2 = np.random.default_rng(seed + 50), np.random.default_rng(seed + 50)
            a, sa = P.atsfft2d(img.x, P.TunerConfig(), 8, g1)
            b, sb = D.atsfft2d_loopsplit(img.x, P.TunerConfig(), 8, g2)
            assert sa == sb and set(a) == set(b)
            ref = O.as_dict(O.atsfft(img.x, O.TunerParams(), 8, seed + 50)[0])
            assert set(b) == set(ref)
            vmax = max([abs(v) for v in ref.values()] + [1e-30])
            assert all(abs(b[q] - v) <= 1e-10 * max(abs(v), 1e-3 * vmax) for q, v in ref.items())
            assert g1.integers(1 << 40) == g2.integers(1 << 40)
    finally:
        dist.destroy_process_group()
