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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_items = 5
    idx = D.batch_shard(n_items, rank, world)
    local = []
    for i in idx:
        img = sparse_image(64, 3, 10 + i, snr_db=25.0)
        (cs, vs), st = O.atsfft(img.x, O.TunerParams(), 4, 20 + i)
        local.append((i, (cs.tolist(), [complex(v) for v in vs], st["detected_k"])))
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    if rank == 0:
        out = [None] * n_items
        for part in gathered:
            for i, r in part:
                out[i] = r
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
