"""The multi-GPU product entry points with TWO ranks (world size 2) on the one
leased GPU: `sfft2d_loopsplit`, `atsfft2d_loopsplit` and `atsfft2d_sharded`
run unchanged in two processes joined by a gloo process group (its
collectives go through host memory, so the ranks' kernels never wait on one
another on the device).  Every rank must return the single-GPU result, and
that result must equal the reference's golden output (fp64: support exact,
values within 1e-10, trajectory exact)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from tests.conftest import fixture_input, golden

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _as_lists(d):
    return [(k, complex(v)) for k, v in d.items()]


def _worker(rank, world, port, out_path):
    import torch.distributed as dist

    import paper_1908_02461_b200 as P
    from paper_1908_02461_b200 import distributed as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        # SFFT loop split: location loops 0,2,4,6 / 1,3,5,7 per rank
        g = golden("c2_sfft")
        x = torch.from_numpy(fixture_input(g)).cuda()
        n, k, loops, b, thr, seed = (int(v) for v in g["cfg"])
        cfg = P.SfftConfig(n=n, k=k, loops=loops, b_bins=b, vote_threshold=thr)
        out["sfft"] = _as_lists(D.sfft2d_loopsplit(x, cfg, seed, precision="fp64"))
        # ATSFFT estimation split (b_estimate = 256 < n: the 8 loops are split)
        g = golden("c4b_00")
        x = torch.from_numpy(fixture_input(g)).cuda()
        gen = np.random.default_rng(int(g["seed"]))
        res, st = D.atsfft2d_loopsplit(x, P.TunerConfig(), 8, gen, precision="fp64")
        out["ats"] = (_as_lists(res), [(bb, c) for bb, c, _ in st.history], st.b_estimate,
                      int(gen.integers(1 << 40)))
        # batch sharding: 4 images, 2 per rank, full list on every rank
        names = ["c4b_00", "c4b_01", "c4b_02", "c4b_03"]
        xs = [torch.from_numpy(fixture_input(golden(nm))).cuda() for nm in names]
        seeds = [int(golden(nm)["seed"]) for nm in names]
        got = D.atsfft2d_sharded(xs, P.TunerConfig(), 8, seeds, concurrency=2, precision="fp64")
        out["sharded"] = [(_as_lists(r), [(bb, c) for bb, c, _ in s.history]) for r, s in got]
        # a NaN seen by one rank's input only: every rank raises ValueError
        xbad = torch.from_numpy(fixture_input(golden("c2_sfft"))).cuda()
        if rank == 1:
            xbad[3, 3] = float("nan")
        cfg1 = P.SfftConfig(n=1024, k=50, loops=1)   # rank 1 owns no location loop
        try:
            D.sfft2d_loopsplit(xbad, cfg1, 5)
            out["nan"] = "returned"
        except ValueError as e:
            out["nan"] = f"ValueError:{e}"
    finally:
        torch.save(out, f"{out_path}.{rank}")
        dist.barrier()
        dist.destroy_process_group()


def _ref(g):
    return dict(zip(map(tuple, g["coords"].tolist()), g["vals"]))


def _close(got_list, g, tol=1e-10):
    got = dict(got_list)
    ref = _ref(g)
    assert list(got) == list(ref)          # the reference's dict order too
    vmax = max([abs(v) for v in ref.values()] + [1e-300])
    for key, v in ref.items():
        assert abs(got[key] - v) <= tol * max(abs(v), 1e-3 * vmax), key


def test_two_ranks_product_entry_points():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1908_02461_b200 as P
    with tempfile.TemporaryDirectory() as td:
        base = os.path.join(td, "res")
        mp.spawn(_worker, args=(2, _free_port(), base), nprocs=2, join=True)
        r0, r1 = torch.load(base + ".0", weights_only=False), torch.load(base + ".1",
                                                                         weights_only=False)
    for key in ("sfft", "ats", "sharded"):
        assert r0[key] == r1[key], key         # every rank ends with the same answer
    _close(r0["sfft"], golden("c2_sfft"))
    g = golden("c4b_00")
    res, hist, b_est, nxt = r0["ats"]
    _close(res, g)
    assert hist == [(int(b), int(c)) for b, c in g["hist"][:, :2]]
    assert b_est == int(g["state"][3]) < 1024
    # the single-GPU call agrees and leaves the Generator where the split does
    gen = np.random.default_rng(int(g["seed"]))
    single, _ = P.atsfft2d(fixture_input(g), P.TunerConfig(), 8, gen)
    assert list(single) == [k for k, _ in res]
    assert int(gen.integers(1 << 40)) == nxt
    for (res_i, hist_i), nm in zip(r0["sharded"], ["c4b_00", "c4b_01", "c4b_02", "c4b_03"]):
        gi = golden(nm)
        _close(res_i, gi)
        assert hist_i == [(int(b), int(c)) for b, c in gi["hist"][:, :2]]
    assert r1["nan"] == "ValueError:matrix contains NaN or Inf"
    assert r0["nan"].startswith("ValueError:")
