"""Pin the CPU oracle (oracle/sfft_oracle.py) to golden vectors produced by the
real reference (oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import sfft_oracle as O
from tests.conftest import assert_int_array, fixture_input, golden, golden_names


def test_windows_match_reference():
    g = golden("windows")
    meta, space, freq = g["meta"], g["space"], g["freq"]
    off = 0
    for n, b, dstop, dpass, support, half, phw in meta:
        n, b = int(n), int(b)
        w = O.window(n, b, dstop, dpass)
        assert w.support == int(support) and w.half == int(half) and w.pass_hw == int(phw)
        np.testing.assert_allclose(w.space, space[off:off + n], rtol=0, atol=1e-13 * n)
        np.testing.assert_allclose(w.freq, freq[off:off + n], rtol=0, atol=1e-13)
        off += n


def test_window_supports_16384():
    g = golden("windows_16384")
    for row in g["meta"]:
        n, b, support, half = (int(v) for v in row[:4])
        if b > 1024:
            continue  # large-b windows take long in pure Python; pinned by the golden meta
        w = O.window(n, b, 1e-8, 1e-3)
        assert (w.support, w.half) == (support, half)
        assert abs(w.space.sum() - row[4]) <= 1e-9 * abs(row[4])


def test_binned_spectrum_matches_reference():
    g = golden("binned")
    for idx in range(int(g["ncases"])):
        n, b, dstop, dpass, seed = g[f"cfg{idx}"]
        n, b = int(n), int(b)
        if f"x{idx}" in g:
            x = g[f"x{idx}"]
        else:
            r = np.random.default_rng(int(seed))
            x = (r.normal(size=(n, n)) + 1j * r.normal(size=(n, n))).astype(np.complex64)
        p = O.make_perm(n, *[int(v) for v in g[f"perm{idx}"][:4]])
        spec = O.bucket_spectrum(O.as_c128(x), p, O.window(n, b, dstop, dpass), b)
        ref = g[f"spec{idx}"]
        assert np.abs(spec - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max())


def test_local_maxima_match_reference():
    g = golden("localmax")
    for i in range(int(g["ngrids"])):
        cnt, coords = O.local_maxima(g[f"grid{i}"], 1e-3)
        assert cnt == int(g[f"count{i}"])
        np.testing.assert_array_equal(coords, g[f"coords{i}"])


def _check_sfft(name):
    g = golden(name)
    x = fixture_input(g)
    n, k, loops, b, thr, seed = (int(v) for v in g["cfg"])
    cfg = O.sfft_params(n, k, loops=loops, b_bins=b, vote_threshold=thr,
                        prune_rel=0.0 if name == "sfft_n16_bn" else 1e-3)
    (cs, vs), trace = O.sfft(x, cfg, seed, return_trace=True)
    rows = [[p.s1, p.s2, p.t1, p.t2, p.s1i, p.s2i] for p in trace["loc_perms"] + trace.get("est_perms", [])]
    np.testing.assert_array_equal(np.array(rows)[: len(rows)], g["perms"][: len(rows)])
    voted = np.stack([trace["keys"] // n, trace["keys"] % n], axis=1) if trace["keys"].size else \
        np.empty((0, 2), np.int64)
    np.testing.assert_array_equal(voted, g["voted"])
    assert {tuple(c) for c in cs.tolist()} == {tuple(c) for c in g["coords"].tolist()}
    ref = dict(zip(map(tuple, g["coords"].tolist()), g["vals"]))
    for c, v in zip(map(tuple, cs.tolist()), vs):
        assert abs(v - ref[c]) <= 1e-10 * max(1.0, abs(ref[c]))


@pytest.mark.parametrize("name", ["c1_sfft", "sfft_n64_k4", "sfft_n128_k4", "sfft_n16_bn",
                                  "sfft_zero", "sfft_n256_noisy", "sfft_n2048_k2_b64"])
def test_sfft_matches_reference(name):
    _check_sfft(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2_sfft", "c3_sfft"])
def test_sfft_large_matches_reference(name):
    _check_sfft(name)


def _check_ats(name):
    g = golden(name)
    x = fixture_input(g)
    t = g["tuner"]
    cfg = O.TunerParams(b0=int(t[0]), eps1=t[1], eps2=t[2], delta1=t[3], delta2=t[4],
                        max_iters=None if t[5] < 0 else int(t[5]), mag_floor=t[6])
    (cs, vs), state, trace = O.atsfft(x, cfg, int(g["est_loops"]), int(g["seed"]), return_trace=True)
    hist = np.array([(b, c, np.nan if r is None else r) for b, c, r in state["history"]],
                    dtype=np.float64).reshape(-1, 3)
    np.testing.assert_array_equal(hist[:, :2], g["hist"][:, :2])
    np.testing.assert_allclose(hist[:, 2], g["hist"][:, 2], rtol=1e-15, atol=0, equal_nan=True)
    st = g["state"]
    assert [int(state["converged"]), state["detected_k"], state["b_detect"], state["b_estimate"],
            state["vote_passes"]] == [int(v) for v in st]
    vc, vt = trace["votes"]
    assert_int_array(vc[:, 0] * x.shape[0] + vc[:, 1] if vc.size else vc.reshape(-1), g, "vote_keys")
    assert_int_array(vt, g, "vote_tallies")
    assert {tuple(c) for c in cs.tolist()} == {tuple(c) for c in g["coords"].tolist()}
    ref = dict(zip(map(tuple, g["coords"].tolist()), g["vals"]))
    vmax = max([abs(v) for v in g["vals"]], default=1.0)
    for c, v in zip(map(tuple, cs.tolist()), vs):
        assert abs(v - ref[c]) <= 1e-10 * max(abs(ref[c]), 1e-3 * vmax)


@pytest.mark.parametrize("name", ["ats_n256_k8", "ats_n64_k1_b8", "ats_dc", "ats_zero",
                                  "ats_noconv", "ats_n256_20db", "ats_n128_15db", "ats_n512_25db"])
def test_atsfft_matches_reference(name):
    _check_ats(name)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2_ats", "c4_k20", "c4_k200", "c3_ats", "c3_ats_clean"])
def test_atsfft_large_matches_reference(name):
    _check_ats(name)


def test_golden_inventory():
    # every fixture the generator writes is exercised by some test here
    names = set(golden_names(""))
    assert {"windows", "binned", "localmax", "c1_sfft", "ats_n256_k8"} <= names
