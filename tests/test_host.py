"""CPU tests of the host-side mirror (configs, permutations, windows, coordinate
maps, tuner rules) and of the C-ABI library surface (loads, exports every
symbol include/sfft2d_b200.h declares).  No GPU needed."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1908_02461_b200 as P
from paper_1908_02461_b200 import _native, engine, hashing, tuner
from oracle import sfft_oracle as O
from tests.conftest import ROOT, golden


def test_library_exports_header_symbols():
    from paper_1908_02461_b200.build import build
    build()
    header = open(os.path.join(ROOT, "include", "sfft2d_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int64_t|int|void|double|const char\*)\s+(sfft2d_\w+)\s*\(", header, re.M))
    assert declared == set(_native.EXPORTS)
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.load_library().sfft2d_abi_version() == 3


def test_struct_layouts_match_header():
    # the ctypes mirrors must have the C sizes (checked against the header's field lists)
    assert ctypes.sizeof(_native.Perm) == 48
    assert ctypes.sizeof(_native.SfftCfg) == 6 * 4 + 4 * 8
    assert ctypes.sizeof(_native.TunerCfg) == 2 * 4 + 9 * 8
    assert ctypes.sizeof(_native.ResultC) == 8 + 4 + 4 + 8 + 4 + 4


def test_no_device_fails_loudly(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    monkeypatch.setattr(_native, "_contexts", {})
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.sfft2d(np.zeros((16, 16), np.complex64), P.SfftConfig(n=16, k=1), 0)


def test_windows_match_reference_golden():
    g = golden("windows")
    off = 0
    for n, b, dstop, dpass, support, half, phw in g["meta"]:
        n, b = int(n), int(b)
        w = hashing.build_flat_window(n, b, dstop, delta_pass=dpass)
        assert (w.support_w, w.half_support, w.pass_halfwidth) == (int(support), int(half), int(phw))
        np.testing.assert_allclose(w.space_1d, g["space"][off:off + n], rtol=0, atol=1e-13 * n)
        np.testing.assert_allclose(w.freq_1d, g["freq"][off:off + n], rtol=0, atol=1e-13)
        off += n


def test_window_supports_16384_match_reference():
    for row in golden("windows_16384")["meta"]:
        n, b, support, half = (int(v) for v in row[:4])
        w = hashing.build_flat_window(n, b, 1e-8, delta_pass=1e-3)
        assert (w.support_w, w.half_support) == (support, half)


def test_host_tables_layout():
    space, freq, tw = hashing.host_tables(64, 1e-3, 1e-8)
    assert space.shape == (7, 64) and freq.shape == (7, 64) and tw.shape == (128,)
    np.testing.assert_array_equal(space[6], np.ones(64))          # b == n: all-pass
    np.testing.assert_array_equal(space[4], hashing.build_flat_window(64, 16, 1e-8, delta_pass=1e-3).space_1d)
    t = tw.view(np.complex128)
    np.testing.assert_array_equal(t, np.exp(-2j * np.pi * np.arange(64) / 64))


def test_permutation_draws_match_oracle():
    a, b = np.random.default_rng(3), np.random.default_rng(3)
    for _ in range(50):
        p, q = hashing.draw_permutation(256, a), O.draw_perm(256, b)
        assert (p.sigma1, p.sigma2, p.tau1, p.tau2, p.sigma1_inv, p.sigma2_inv) == \
            (q.s1, q.s2, q.t1, q.t2, q.s1i, q.s2i)


def test_permutation_params():
    p = hashing.PermutationParams(16, 3, 5, 7, 2)
    assert (p.sigma1_inv, p.sigma2_inv) == (11, 13)
    with pytest.raises(ValueError):
        hashing.PermutationParams(16, 2, 5, 0, 0)


def test_config_validation_mirrors_reference():
    assert engine.default_bins(256, 8) == 32
    assert engine.default_bins(2048, 8) == 32
    assert engine.default_bins(256, 16) == 64
    assert engine.default_bins(256, 2) == 16
    with pytest.raises(P.ConfigurationError):
        P.SfftConfig(n=16, k=200)
    with pytest.raises(P.ConfigurationError):
        P.SfftConfig(n=64, k=2, loops=4, vote_threshold=5)
    assert P.SfftConfig(n=64, k=2, loops=8).vote_threshold == 4
    assert P.SfftConfig(n=64, k=2, loops=5).vote_threshold == 3
    with pytest.raises(P.ConfigurationError):
        P.TunerConfig(delta1=0.05, delta2=0.02)
    with pytest.raises(P.ConfigurationError):
        P.TunerConfig(eps1=1.5)
    assert issubclass(P.ConfigurationError, ValueError)


@pytest.mark.parametrize("r,expected", [(0.0, 32), (0.019, 32), (0.02, 64), (0.049, 64),
                                        (0.05, 128), (1.0, 128)])
def test_update_bins_branch_table(r, expected):
    assert P.update_bins(64, r, P.TunerConfig(), 4096) == expected


def test_update_bins_matches_oracle_exhaustive():
    cfg, ocfg = P.TunerConfig(), O.TunerParams()
    for n in (16, 256, 4096):
        b = 4
        while b <= n:
            for r in (0.0, 0.019, 0.02, 0.049, 0.05, 1.0, float("inf")):
                assert P.update_bins(b, r, cfg, n) == O.next_bins(b, r, ocfg, n)
            b *= 2


def test_hash_unhash_round_trip():
    rng = np.random.default_rng(1)
    n, b = 32, 8
    for _ in range(5):
        p = hashing.draw_permutation(n, rng)
        for i in range(n):
            for j in range(n):
                bi, bj = hashing.hash_coord(i, j, p, n, b)
                c = hashing.unhash_bin(bi, bj, p, n, b)
                assert ((c[:, 0] == i) & (c[:, 1] == j)).any()
                oi, oj = hashing.offset_coord(i, j, p, n, b)
                assert abs(oi) <= n // (2 * b) and abs(oj) <= n // (2 * b)


def test_unhash_matches_oracle_expand():
    rng = np.random.default_rng(2)
    for n, b in ((64, 4), (64, 16), (64, 64), (256, 32)):
        p = hashing.draw_permutation(n, rng)
        q = O.make_perm(n, p.sigma1, p.sigma2, p.tau1, p.tau2)
        for bi, bj in ((0, 0), (b - 1, 3 % b), (b // 2, b - 1)):
            keys = O.preimage_keys(np.array([bi]), np.array([bj]), q, n, b, expand=1)
            c = hashing.unhash_bin(bi, bj, p, n, b, expand=1)
            np.testing.assert_array_equal(c[:, 0] * n + c[:, 1], keys)


def test_generator_is_deterministic_and_noisy():
    a = P.sparse_image(64, 5, 3, snr_db=20.0)
    b = P.sparse_image(64, 5, 3, snr_db=20.0)
    np.testing.assert_array_equal(a.x, b.x)
    assert a.x.dtype == np.complex64 and len(set(zip(a.rows, a.cols))) == 5
    c = P.sparse_image(256, 40, 4, cluster_frac=0.2, snr_db=None, dtype=np.complex128)
    near = ((c.rows + 32) % 256 < 64) & ((c.cols + 32) % 256 < 64)
    assert near.sum() >= 8
    spec = np.fft.fft2(c.x)
    np.testing.assert_allclose(spec[c.rows, c.cols], c.coeffs, atol=1e-9)


def test_error_metric():
    assert P.error_metric({(0, 0): 1.0}, {(0, 0): 1.0}, 1) == 0.0
    assert P.error_metric({}, {}, 0) == 0.0
    assert P.error_metric({(1, 1): 1.0}, {}, 0) == float("inf")


def test_every_kernel_waits_on_its_predecessor():
    """Every launch goes through cudaLaunchKernelEx with programmatic stream
    serialization, so every kernel must execute griddepcontrol.wait
    (pdl_wait) before touching memory its predecessor wrote."""
    import glob
    import re
    csrc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "paper_1908_02461_b200", "csrc")
    missing = []
    for path in sorted(glob.glob(os.path.join(csrc, "*.cuh")) + glob.glob(os.path.join(csrc, "*.cu"))):
        src = open(path).read()
        for m in re.finditer(r"__global__\b", src):
            open_brace = src.index("{", m.end())
            name = re.findall(r"(\w+)\s*\(", src[m.end():open_brace])
            name = [n for n in name if n != "__launch_bounds__"]
            body = src[open_brace:open_brace + 400]
            first_stmt = body.split(";")[0]
            if "pdl_wait()" not in first_stmt:
                missing.append(f"{os.path.basename(path)}:{name[0] if name else '?'}")
    assert not missing, missing


def test_generator_reconciled_after_speculative_draw():
    # a permutation drawn ahead (speculative fold) but never consumed must not
    # advance the caller's Generator past where the reference leaves it
    from paper_1908_02461_b200.hashing import draw_permutation
    from paper_1908_02461_b200.tuner import reconcile_generator
    n, used = 4096, 11
    g = np.random.default_rng(123)
    snap = g.bit_generator.state
    for _ in range(used + 1):
        draw_permutation(n, g)
    reconcile_generator(g, snap, n, used + 1, used)
    ref = np.random.default_rng(123)
    for _ in range(used):
        draw_permutation(n, ref)
    assert g.bit_generator.state == ref.bit_generator.state
    # nothing to undo when every draw was consumed
    before = g.bit_generator.state
    reconcile_generator(g, snap, n, used, used)
    assert g.bit_generator.state == before


@pytest.mark.parametrize("shape", [(0, 0), (8,), (4, 8), (6, 6), (3, 3), (2, 4, 4), (1, 2)])
def test_bad_shapes_rejected_like_reference(shape):
    # corefft.as_complex_matrix (corefft.py:38-51): square, power-of-two sides only
    from paper_1908_02461_b200._tensors import host_image
    x = np.zeros(shape, dtype=np.complex64)
    with pytest.raises(ValueError):
        O.as_c128(x)
    with pytest.raises(ValueError):
        host_image(x)


@pytest.mark.parametrize("dtype", [np.int32, np.float32, np.float64, np.complex64, np.complex128])
def test_numeric_inputs_accepted_like_reference(dtype):
    from paper_1908_02461_b200._tensors import host_image
    x = (np.arange(16).reshape(4, 4) % 5).astype(dtype)
    a, code = host_image(x)
    ref = O.as_c128(x)
    assert a.shape == (4, 4) and np.array_equal(a.astype(np.complex128), ref)
    assert code == (_native.C64 if dtype == np.complex64 else _native.C128)


def test_check_window_rejects_foreign_weights():
    import dataclasses
    from paper_1908_02461_b200 import hashing as H
    w = H.build_flat_window(256, 16, 1e-8, delta_pass=1e-3)
    H.check_window(w)
    H.check_window(H.all_pass_window(256))
    with pytest.raises(ValueError, match="window weights differ"):
        H.check_window(dataclasses.replace(w, space_1d=w.space_1d * (1 + 1e-9)))
    with pytest.raises(ValueError, match="window weights differ"):
        H.check_window(dataclasses.replace(w, freq_1d=np.roll(w.freq_1d, 1)))


def test_batch_detects_shared_generators():
    from paper_1908_02461_b200.batch import _shared_generators
    g = np.random.default_rng(1)
    assert _shared_generators([g, np.random.default_rng(1), g])
    assert not _shared_generators([g, np.random.default_rng(1), 3, 3])


@pytest.mark.parametrize("seed", [0, 1, 12, 2**40 + 3, 2**62 + 12345])
@pytest.mark.parametrize("n", [16, 256, 4096, 16384])
def test_native_sfft_streams_match_numpy(seed, n):
    # engine.py:266-280 restated natively (numpy SeedSequence + PCG64 in
    # csrc/npyrng.h): the 2L child permutations and the caller's Generator
    # advance are numpy's own (host-only entry point, no GPU needed)
    lib = _native.load_library()
    loops = 8
    g1, g2 = np.random.default_rng(seed), np.random.default_rng(seed)
    out = (_native.Perm * (2 * loops))()
    assert lib.sfft2d_sfft_draw_perms(g1.bit_generator.ctypes.bit_generator.value, n, loops,
                                      out) == 0
    kids = [np.random.default_rng(int(g2.integers(2**63))) for _ in range(2 * loops)]
    want = [hashing.draw_permutation(n, k) for k in kids]
    got = [(o.sigma1, o.sigma2, o.tau1, o.tau2, o.sigma1_inv, o.sigma2_inv) for o in out]
    assert got == [(p.sigma1, p.sigma2, p.tau1, p.tau2, p.sigma1_inv, p.sigma2_inv) for p in want]
    assert g1.integers(1 << 40) == g2.integers(1 << 40)
