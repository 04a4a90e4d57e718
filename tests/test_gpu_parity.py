"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the
reference's golden vectors.

Tolerances (north star): coordinates / counts / votes / trajectories exact;
values within 1e-10 relative in fp64 mode and 1e-4 relative in fp32 mode,
"relative" meaning |a - b| <= tol * max(|b|, 1e-3 * max|b|) (the 1e-3 floor
is the reference's own prune level, engine.py:249).
"""

import numpy as np
import pytest

import paper_1908_02461_b200 as P
from oracle import sfft_oracle as O
from tests.conftest import assert_int_array, fixture_input, golden

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-10, "fp32": 1e-4}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _close_values(got: dict, ref: dict, tol: float):
    """Same support and values within tol.  fp32 only: a coefficient may be
    on one side alone when its magnitude sits within the value tolerance of a
    selection boundary of the reference's float64 median (the prune level
    prune_rel * max|v|, engine.py:249, or the smallest kept magnitude of a
    top-k cut): the fp32 median is within tol of the float64 one, so the
    comparison against that boundary can go either way — in noise-dominated
    outputs with tens of thousands of coefficients (c5 k=1024) a few do."""
    only_got, only_ref = set(got) - set(ref), set(ref) - set(got)
    if tol < 1e-6 or not ref:
        assert not only_got and not only_ref, (len(only_got), len(only_ref))
    if not ref:
        return
    vmax = max(abs(v) for v in ref.values())
    if only_got or only_ref:
        bounds = [1e-3 * vmax, min(abs(v) for v in ref.values())]
        for key in only_got | only_ref:
            m = abs(got[key]) if key in got else abs(ref[key])
            assert any(abs(m - b) <= 2 * tol * b for b in bounds), (key, m, bounds)
        assert len(only_got) + len(only_ref) <= max(2, len(ref) // 10000), (len(only_got), len(only_ref))
    worst = 0.0
    for key, v in ref.items():
        if key not in got:
            continue
        err = abs(got[key] - v) / max(abs(v), 1e-3 * vmax, 1e-300)
        worst = max(worst, err)
    assert worst <= tol, worst
    common = [key for key in got if key in ref]
    _check_order(common, {key: ref[key] for key in ref if key in got}, tol)


def _check_order(got_keys: list, ref: dict, tol: float):
    """The dict's iteration order is the reference's: row-major (i, j), or
    lexsort(-|v|, i, j) after a top-k cut (engine.py:245-253).  Row-major
    order must match exactly; in the magnitude order two entries may only
    trade places when their reference magnitudes are equal within the value
    tolerance (a near-tie of the sort key: unit-magnitude noiseless spectra
    differ only in the last ulps of |v|, which no two float64 codes share)."""
    ref_keys = list(ref)
    if got_keys == ref_keys:
        return
    assert ref_keys != sorted(ref_keys), "row-major order differs from the reference"
    pos = {key: i for i, key in enumerate(ref_keys)}
    mags = [abs(ref[key]) for key in got_keys]
    for i, key in enumerate(got_keys):
        j = pos[key]
        if i != j:   # displaced: its magnitude ties (within tol) the one it displaced
            assert abs(mags[i] - abs(ref[ref_keys[i]])) <= 2 * tol * max(mags[i], 1e-300), key


def _ref_dict(g):
    return dict(zip(map(tuple, g["coords"].tolist()), g["vals"]))


# ------------------------------------------------------------- building blocks
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_binned_spectrum_vs_reference(precision):
    g = golden("binned")
    for idx in range(int(g["ncases"])):
        n, b, dstop, dpass, seed = g[f"cfg{idx}"]
        n, b = int(n), int(b)
        if f"x{idx}" in g:
            x = g[f"x{idx}"]
        else:
            r = np.random.default_rng(int(seed))
            x = (r.normal(size=(n, n)) + 1j * r.normal(size=(n, n))).astype(np.complex64)
        row = [int(v) for v in g[f"perm{idx}"]]
        p = P.PermutationParams(n, *row[:4])
        win = P.build_flat_window(n, b, dstop, delta_pass=dpass)
        spec = P.binned_spectrum(x, p, win, b, precision=precision).spectrum
        ref = g[f"spec{idx}"]
        err = np.abs(spec - ref).max() / np.abs(ref).max()
        assert err <= (1e-12 if precision == "fp64" else 2e-6), (idx, n, b, err)


def test_binned_spectrum_multi_loop_shares_read():
    rng = np.random.default_rng(7)
    for n, b in ((256, 16), (1024, 64), (512, 512), (2048, 1024)):
        x = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)
        win = P.build_flat_window(n, b, 1e-8, delta_pass=1e-3)
        perms = [P.draw_permutation(n, rng) for _ in range(5)]
        many = P.binned_spectrum(x, perms, win, b).spectrum
        ow = O.window(n, b, 1e-8, 1e-3)
        a = O.as_c128(x)
        for i, p in enumerate(perms):
            ref = O.bucket_spectrum(a, O.make_perm(n, p.sigma1, p.sigma2, p.tau1, p.tau2), ow, b)
            assert np.abs(many[i] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_count_local_maxima_vs_reference():
    g = golden("localmax")
    for i in range(int(g["ngrids"])):
        grid = g[f"grid{i}"]          # includes non-power-of-two sides
        cnt, coords = P.count_local_maxima(grid, 1e-3)
        assert cnt == int(g[f"count{i}"])
        np.testing.assert_array_equal(coords, g[f"coords{i}"])


def test_count_local_maxima_random_vs_oracle():
    rng = np.random.default_rng(11)
    for b in (4, 5, 6, 8, 12, 64, 100, 256, 300, 1024):
        grid = rng.normal(size=(b, b)) + 1j * rng.normal(size=(b, b))
        cnt, coords = P.count_local_maxima(grid, 1e-3)
        ocnt, ocoords = O.local_maxima(grid, 1e-3)
        assert cnt == ocnt
        np.testing.assert_array_equal(coords, ocoords)


def test_top_bins_ties_lowest_index():
    import ctypes
    import torch
    from paper_1908_02461_b200 import _native
    ctx = _native.context()
    rng = np.random.default_rng(3)
    for b, num, nseg in ((16, 5, 3), (64, 100, 2), (256, 2000, 4), (8, 64, 1)):
        grids = (rng.integers(0, 4, size=(nseg, b, b)) * (1 + 1j)).astype(np.complex128)
        t = torch.from_numpy(grids).cuda()
        out = torch.empty((nseg, num), dtype=torch.int32, device="cuda")
        ctx.check(ctx.lib.sfft2d_top_bins(ctx.handle, t.data_ptr(), b, nseg, num, 1,
                                          out.data_ptr(), torch.cuda.current_stream().cuda_stream))
        got = out.cpu().numpy()
        for s in range(nseg):
            want = np.sort(O.top_bins(grids[s], num))
            np.testing.assert_array_equal(got[s], want)


# ------------------------------------------------------------- Algorithm 1
SFFT_CASES = ["c1_sfft", "sfft_n64_k4", "sfft_n128_k4", "sfft_n16_bn", "sfft_zero",
              "sfft_n256_noisy", "sfft_n2048_k2_b64", "c2_sfft", "c3_sfft"]


def _sfft_cfg(g, name):
    n, k, loops, b, thr, seed = (int(v) for v in g["cfg"])
    cfg = P.SfftConfig(n=n, k=k, loops=loops, b_bins=b, vote_threshold=thr,
                       prune_rel=0.0 if name == "sfft_n16_bn" else 1e-3)
    return cfg, seed


@pytest.mark.parametrize("name", SFFT_CASES)
def test_sfft_fp64_vs_reference(name):
    g = golden(name)
    x = fixture_input(g)
    cfg, seed = _sfft_cfg(g, name)
    out = P.sfft2d(x, cfg, seed, precision="fp64")
    _close_values(out, _ref_dict(g), TOL["fp64"])


@pytest.mark.parametrize("name", ["c1_sfft", "sfft_n128_k4", "sfft_n2048_k2_b64", "c2_sfft", "c3_sfft"])
def test_sfft_fp32_vs_reference(name):
    g = golden(name)
    x = fixture_input(g)
    cfg, seed = _sfft_cfg(g, name)
    out = P.sfft2d(x, cfg, seed, precision="fp32")
    _close_values(out, _ref_dict(g), TOL["fp32"])


def test_sfft_seeded_determinism_and_rng_advance():
    sig = P.planted_image(128, 4, 77)
    a = P.sfft2d(sig.x, P.SfftConfig(n=128, k=4), 42)
    b = P.sfft2d(sig.x, P.SfftConfig(n=128, k=4), 42)
    assert a == b
    g1, g2 = np.random.default_rng(5), np.random.default_rng(5)
    P.sfft2d(sig.x, P.SfftConfig(n=128, k=4), g1)
    O.sfft(sig.x, O.sfft_params(128, 4), g2)
    assert g1.integers(1 << 30) == g2.integers(1 << 30)


def test_sfft_wrong_side_and_nan():
    with pytest.raises(P.ConfigurationError):
        P.sfft2d(np.zeros((32, 32)), P.SfftConfig(n=64, k=2), 0)
    x = np.zeros((64, 64), np.complex64)
    x[3, 3] = np.nan
    with pytest.raises(ValueError, match="NaN"):
        P.sfft2d(x, P.SfftConfig(n=64, k=2), 0)


def test_sfft_many_loops_groups():
    # L > 8: votes go through per-group bitmasks + counters
    sig = P.planted_image(256, 6, 5)
    cfg = P.SfftConfig(n=256, k=6, loops=11)
    o = O.sfft(sig.x, O.sfft_params(256, 6, loops=11), 9)
    _close_values(P.sfft2d(sig.x, cfg, 9), O.as_dict(o), TOL["fp64"])


# ------------------------------------------------------------- Algorithm 2
ATS_CASES = ["ats_n256_k8", "ats_n64_k1_b8", "ats_dc", "ats_zero", "ats_noconv", "ats_n256_20db",
             "ats_n128_15db", "ats_n512_25db", "c2_ats", "c4_k20", "c4_k200", "c3_ats_clean",
             "c3_ats"]


def _tuner(g):
    t = g["tuner"]
    return P.TunerConfig(b0=int(t[0]), eps1=float(t[1]), eps2=float(t[2]), delta1=float(t[3]),
                         delta2=float(t[4]), max_tuning_iters=None if t[5] < 0 else int(t[5]),
                         mag_floor=float(t[6]))


# Noiseless planted spectra put isolated coefficients exactly half a bin from
# two bin centres at even w: the two bins' magnitudes are then equal up to
# roundoff and the strict ">" of count_local_maxima is decided by the last ulp,
# which differs between any two float64 implementations (numpy's own result
# depends on the CPU's SIMD path: FMA complex multiply, SIMD abs).  For those
# cases the trajectory is not a well-defined parity target; the recovered
# support and values are (and must match exactly / within tolerance).
NOISELESS = {"ats_n256_k8", "ats_n64_k1_b8", "ats_dc", "ats_noconv", "c3_ats_clean"}


def _near_tie_pass(x, g, t, rel=1e-12):
    """Whether tuner pass t of the reference trajectory (its B, its t-th
    permutation draw) holds a magnitude near-tie that decides a count: a bin
    at or above the floor within `rel` of its largest 8-neighbour, or a bin
    within `rel` of the floor itself."""
    O.FAST = True
    try:
        a = O.as_c128(x)
        n = a.shape[0]
        tc = _tuner(g)
        gen = np.random.default_rng(int(g["seed"]))
        perms = [O.draw_perm(n, gen) for _ in range(t + 1)]
        b = int(g["hist"][t, 0])
        win = O.cached_window(n, b, tc.window_delta_stop, tc.window_delta_pass)
        m = np.abs(O.bucket_spectrum(a, perms[t], win, b))
    finally:
        O.FAST = False
    top = m.max()
    if top == 0:
        return False
    nb = np.max([np.roll(m, (du, dv), axis=(0, 1)) for du in (-1, 0, 1) for dv in (-1, 0, 1)
                 if du or dv], axis=0)
    live = m >= tc.mag_floor * top * (1 - rel)
    tie_nb = np.any(live & (np.abs(m - nb) <= rel * m))
    tie_floor = np.any(np.abs(m - tc.mag_floor * top) <= rel * top)
    return bool(tie_nb or tie_floor)


def _check_state(state, g, name="", precision="fp64", x=None):
    if name in NOISELESS and precision == "fp64":
        # exact trajectory unless the first differing pass holds a near-tie
        # that the last ulp decides (proven per case from the oracle's grids)
        got = [(b, c) for b, c, _ in state.history]
        ref = [(int(b), int(c)) for b, c in g["hist"][:, :2]]
        if got == ref:
            return
        t = next(i for i, (u, v) in enumerate(zip(got, ref)) if u != v) if any(
            u != v for u, v in zip(got, ref)) else min(len(got), len(ref)) - 1
        assert got[t][0] == ref[t][0], (t, got[t], ref[t])   # same B: only a count flips
        assert x is not None and _near_tie_pass(x, g, t), (name, t, got[t], ref[t])
        return
    if name in NOISELESS:
        return
    if precision == "fp32":
        # fp32 magnitudes: the bin trajectory must match; a count may differ by
        # a near-tie flip among millions of noise bins (tolerance 1e-4 relative)
        got = [(b, c) for b, c, _ in state.history]
        ref = [(int(b), int(c)) for b, c in g["hist"][:, :2]]
        assert [b for b, _ in got] == [b for b, _ in ref]
        for (_, c1), (_, c2) in zip(got, ref):
            assert abs(c1 - c2) <= 1e-4 * max(c2, 1), (c1, c2)
        return
    hist = np.array([(b, c, np.nan if r is None else r) for b, c, r in state.history],
                    dtype=np.float64).reshape(-1, 3)
    np.testing.assert_array_equal(hist[:, :2], g["hist"][:, :2])
    np.testing.assert_array_equal(np.isnan(hist[:, 2]), g["hist_none"])
    np.testing.assert_allclose(hist[:, 2], g["hist"][:, 2], rtol=1e-15, equal_nan=True)
    st = [int(v) for v in g["state"]]
    assert [int(state.converged), state.detected_k, state.b_detect, state.b_estimate,
            state.vote_passes] == st


@pytest.mark.parametrize("name", ATS_CASES)
def test_atsfft_fp64_vs_reference(name):
    g = golden(name)
    x = fixture_input(g)
    out, state = P.atsfft2d(x, _tuner(g), int(g["est_loops"]), int(g["seed"]), precision="fp64")
    _check_state(state, g, name, x=x)
    _close_values(out, _ref_dict(g), TOL["fp64"])


@pytest.mark.parametrize("name", ["ats_n256_20db", "ats_n512_25db", "c2_ats", "c4_k200", "c3_ats"])
def test_detect_sparsity_votes_vs_reference(name):
    g = golden(name)
    x = fixture_input(g)
    state, (coords, tallies) = P.detect_sparsity(x, _tuner(g), int(g["seed"]))
    n = x.shape[0]
    assert_int_array(coords[:, 0] * n + coords[:, 1], g, "vote_keys")
    assert_int_array(tallies, g, "vote_tallies")


@pytest.mark.parametrize("name", ["ats_n256_20db", "ats_n512_25db", "c2_ats", "c4_k20", "c3_ats"])
def test_atsfft_fp32_vs_reference(name):
    g = golden(name)
    x = fixture_input(g)
    out, state = P.atsfft2d(x, _tuner(g), int(g["est_loops"]), int(g["seed"]), precision="fp32")
    _check_state(state, g, name, "fp32")
    _close_values(out, _ref_dict(g), TOL["fp32"])


def test_atsfft_generator_advance_matches_oracle():
    img = P.sparse_image(256, 8, 300, snr_db=25.0)
    g1, g2 = np.random.default_rng(400), np.random.default_rng(400)
    P.atsfft2d(img.x, P.TunerConfig(), 8, g1)
    O.atsfft(img.x, O.TunerParams(), 8, g2)
    assert g1.integers(1 << 40) == g2.integers(1 << 40)


def test_atsfft_generator_advance_with_speculative_fold():
    # N = 2048: B >= 512 passes fold the next pass's 2B grid early (its
    # permutation drawn ahead); results and the caller's Generator must match
    img = P.sparse_image(2048, 30, 71, snr_db=20.0)
    g1, g2 = np.random.default_rng(72), np.random.default_rng(72)
    out, state = P.atsfft2d(img.x, P.TunerConfig(), 8, g1)
    (cs, vs), ostate = O.atsfft(img.x, O.TunerParams(), 8, g2)
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    assert any(b >= 512 for b, _, _ in state.history)
    _close_values(out, O.as_dict((cs, vs)), TOL["fp64"])
    assert g1.integers(1 << 40) == g2.integers(1 << 40)


def test_atsfft_device_tensor_input_matches_numpy():
    import torch
    g = golden("c2_ats")
    x = fixture_input(g)
    a, sa = P.atsfft2d(x, _tuner(g), 8, 11)
    b, sb = P.atsfft2d(torch.from_numpy(x).cuda(), _tuner(g), 8, 11)
    assert a == b and sa == sb


@pytest.mark.parametrize("seed", range(6))
def test_atsfft_random_noisy_vs_oracle(seed):
    # fresh seeded cases beyond the golden set: exact trajectory + support, fp64 values
    n = [128, 256, 512][seed % 3]
    img = P.sparse_image(n, 5 + 7 * seed, 100 + seed, snr_db=[15.0, 20.0, 30.0][seed % 3],
                         magnitude="loguniform" if seed % 2 else "unit")
    (cs, vs), ostate = O.atsfft(img.x, O.TunerParams(), 8, 200 + seed)
    out, state = P.atsfft2d(img.x, P.TunerConfig(), 8, 200 + seed)
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    _close_values(out, O.as_dict((cs, vs)), TOL["fp64"])


@pytest.mark.parametrize("n", [256, 512])
def test_atsfft_wide_tallies_match_oracle(n):
    # max_tuning_iters = 70: tallies can exceed 255, so votes take the 32-bit
    # atomic histogram path instead of the deferred byte tiles
    img = P.sparse_image(n, 9, 500 + n, snr_db=20.0)
    (cs, vs), ostate = O.atsfft(img.x, O.TunerParams(max_iters=70), 8, 9)
    out, state = P.atsfft2d(img.x, P.TunerConfig(max_tuning_iters=70), 8, 9)
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    assert state.vote_passes == ostate["vote_passes"]
    _close_values(out, O.as_dict((cs, vs)), TOL["fp64"])


def test_atsfft_nan_leaves_generator_untouched():
    x = P.sparse_image(128, 4, 1, snr_db=20.0).x.copy()
    x[5, 7] = np.inf
    g = np.random.default_rng(3)
    before = g.bit_generator.state
    with pytest.raises(ValueError, match="NaN or Inf"):
        P.atsfft2d(x, P.TunerConfig(), 8, g)
    assert g.bit_generator.state == before


def test_atsfft_generator_advance_on_configuration_error():
    # detected_k large vs the clamped estimation grid: reference raises after detection
    img = P.sparse_image(64, 40, 2, snr_db=5.0)
    g1, g2 = np.random.default_rng(8), np.random.default_rng(8)
    try:
        O.atsfft(img.x, O.TunerParams(), 8, g2)
        ref_err = None
    except ValueError as e:
        ref_err = e
    try:
        P.atsfft2d(img.x, P.TunerConfig(), 8, g1)
        err = None
    except ValueError as e:
        err = e
    assert (ref_err is None) == (err is None)
    assert g1.integers(1 << 40) == g2.integers(1 << 40)


def test_batch_concurrent_equals_sequential():
    imgs = [P.sparse_image(512, 10 + i, 40 + i, snr_db=25.0, magnitude="loguniform") for i in range(6)]
    xs = [im.x for im in imgs]
    seq = [P.atsfft2d(x, P.TunerConfig(), 8, 100 + i) for i, x in enumerate(xs)]
    par = P.atsfft2d_batch(xs, P.TunerConfig(), 8, [100 + i for i in range(6)], concurrency=3)
    for (a, sa), (b, sb) in zip(seq, par):
        assert a == b and sa == sb
    s1 = [P.sfft2d(x, P.SfftConfig(n=512, k=12), 7) for x in xs]
    s2 = P.sfft2d_batch(xs, P.SfftConfig(n=512, k=12), [7] * 6, concurrency=3)
    assert s1 == s2


@pytest.mark.parametrize("n,precision", [(8192, "fp32"), (8192, "fp64"), (16384, "fp32"),
                                         (16384, "fp64")])
def test_large_fft_sides(n, precision):
    # B = N bucket grid with the identity permutation is the dense 2D DFT
    rng = np.random.default_rng(n)
    x = (rng.standard_normal((n, n), dtype=np.float32)
         + 1j * rng.standard_normal((n, n), dtype=np.float32)).astype(np.complex64)
    win = P.all_pass_window(n)
    got = P.binned_spectrum(x, P.identity_permutation(n), win, n, precision=precision).spectrum
    ref = np.fft.fft2(x.astype(np.complex128))   # float64 pocketfft (numpy 2 keeps c64 in single)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < (1e-5 if precision == "fp32" else 1e-12), err


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c5_atsfft_vs_reference(precision):
    # 16384^2: fp64 rows run as 2-CTA clusters (k_fftr_cl2), fp64 B = N local
    # maxima straight from global memory (k_lmax_direct)
    g = golden("c5_ats_k64")
    x = fixture_input(g)
    out, state = P.atsfft2d(x, _tuner(g), int(g["est_loops"]), int(g["seed"]), precision=precision)
    _check_state(state, g, "c5_ats_k64", precision)
    _close_values(out, _ref_dict(g), TOL[precision])


# ------------------------------------------------------------- c4 batch images
C4B = [f"c4b_{i:02d}" for i in range(12)]


@pytest.mark.parametrize("name", C4B)
def test_c4_bench_images_fp64_vs_reference(name):
    # the first 12 images of the bench's c4 batch (k ~ U[20, 200], log-uniform
    # magnitudes, 25 dB): full state + votes-derived support exact
    g = golden(name)
    x = fixture_input(g)
    out, state = P.atsfft2d(x, _tuner(g), int(g["est_loops"]), int(g["seed"]), precision="fp64")
    _check_state(state, g, name)
    _close_values(out, _ref_dict(g), TOL["fp64"])


def test_c4_bench_images_fp32_batch_vs_reference():
    # the same images through the batch API in fp32 (what the bench times)
    gs = [golden(nm) for nm in C4B]
    xs = [fixture_input(g) for g in gs]
    res = P.atsfft2d_batch(xs, P.TunerConfig(), 8, [int(g["seed"]) for g in gs], concurrency=4,
                           precision="fp32")
    for (out, state), g, nm in zip(res, gs, C4B):
        _check_state(state, g, nm, "fp32")
        _close_values(out, _ref_dict(g), TOL["fp32"])


# ------------------------------------------------------------- c5 sparsity sweep
@pytest.mark.parametrize("k", [256, 1024, 4096])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_c5_sweep_vs_reference(k, precision):
    g = golden(f"c5_ats_k{k}")
    x = fixture_input(g)
    out, state = P.atsfft2d(x, _tuner(g), int(g["est_loops"]), int(g["seed"]), precision=precision)
    _check_state(state, g, f"c5_ats_k{k}", precision)
    _close_values(out, _ref_dict(g), TOL[precision])


def test_count_local_maxima_plateaus_and_floor_ties():
    """Small integer magnitudes: plateaus (the strict '>' must reject equal
    neighbours, tuner.py:112-116), bins exactly at the floor (the '>=' of
    tuner.py:111 must keep them), an all-equal grid and an all-zero grid."""
    rng = np.random.default_rng(5)
    for b in (4, 6, 16, 32, 48, 64, 128, 200, 512):
        for floor in (0.25, 0.5, 1.0):
            grid = rng.integers(0, 5, size=(b, b)).astype(np.complex128)   # |.| in {0..4}, peak 4
            cnt, coords = P.count_local_maxima(grid, floor)
            ocnt, ocoords = O.local_maxima(grid, floor)
            assert cnt == ocnt, (b, floor)
            np.testing.assert_array_equal(coords, ocoords)
        for grid in (np.full((b, b), 3.0 + 0j), np.zeros((b, b), np.complex128)):
            cnt, coords = P.count_local_maxima(grid, 1e-3)
            assert cnt == 0 and coords.shape == (0, 2)


@pytest.mark.parametrize("gain_floor", [0.9999, 1.0 - 1e-10, 1.0, 1.0 + 2e-4])
def test_sfft_partially_unusable_loops_match_oracle(gain_floor):
    """gain_floor inside the window's passband (gain 0.999875 at bucket offset
    +-4, 1 - 8e-10 at +-3, exactly 1 inside, for n = 256, B = 32): a loop's
    estimate of a coordinate is usable or not depending on its offset in the
    bucket, so the medians run over loop subsets (and through the reference's
    complex nan mask, engine.py:241-242); above 1 every coordinate is dead and
    the result is empty."""
    n, k = 256, 8
    img = P.sparse_image(n, k, 21, snr_db=30.0, dtype=np.complex128)
    cfg = P.SfftConfig(n=n, k=k, gain_floor=gain_floor)
    got = P.sfft2d(img.x, cfg, 9, precision="fp64")
    want = O.as_dict(O.sfft(img.x, O.sfft_params(n, k, gain_floor=gain_floor), 9))
    assert list(got) == list(want)
    for key, v in want.items():
        assert abs(got[key] - v) <= 1e-10 * max(1.0, abs(v)), (key, got[key], v)


@pytest.mark.parametrize("gain_floor", [0.9999, 1.0 - 1e-10, 1.0 + 2e-4])
def test_atsfft_partially_unusable_loops_match_oracle(gain_floor):
    """Algorithm 2 with mag_floor = 0.2 on a 30 dB image (the noise maxima
    stay below the floor, so detected_k = k and b_estimate = 32 < N: the
    estimation loops go through the window gain; the noise breaks the exact
    ties of a noiseless image, so the trajectory is the reference's) and a
    gain_floor inside the passband: the estimation loops of a coordinate are
    partly unusable and the medians take the reference's complex nan mask."""
    img = P.sparse_image(256, 6, 3, snr_db=30.0, dtype=np.complex128)
    cfg = P.TunerConfig(mag_floor=0.2, gain_floor=gain_floor)
    got, state = P.atsfft2d(img.x, cfg, 8, 4, precision="fp64")
    (cs, vs), ostate = O.atsfft(img.x, O.TunerParams(mag_floor=0.2, gain_floor=gain_floor), 8, 4)
    want = O.as_dict((cs, vs))
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    assert state.b_estimate == ostate["b_estimate"] < 256
    assert list(got) == list(want)
    for key, v in want.items():
        assert abs(got[key] - v) <= 1e-10 * max(1.0, abs(v)), (key, got[key], v)


def _fuzz_compare(got: dict, want: dict):
    """fp64 fuzz comparison: same support, dict order and values (1e-10).  One
    loop estimates every coordinate aliased into a bucket from the same bucket
    value, so such coordinates have magnitudes equal up to the last ulps of
    the phase twist; a top-k cut through a group of them is decided by those
    ulps (numpy's own answer depends on the summation order of its FFT).  A
    coordinate may therefore be on one side alone only when its magnitude
    equals the smallest kept magnitude to 1e-12, and entries may trade places
    in the magnitude order only under the same condition."""
    only = set(got) ^ set(want)
    if only:
        assert len(got) == len(want)
        bound = min(abs(v) for v in want.values())
        for key in only:
            m = abs(got[key]) if key in got else abs(want[key])
            assert abs(m - bound) <= 1e-12 * bound, (key, m, bound)
    common = {key: want[key] for key in want if key in got}
    _check_order([key for key in got if key in common], common, 1e-10)
    vmax = max([abs(v) for v in want.values()] or [1.0])
    for key, v in common.items():
        assert abs(got[key] - v) <= 1e-10 * max(abs(v), 1e-3 * vmax), (key, got[key], v)


def _fuzz_cases():
    rng = np.random.default_rng(2024)
    cases = []
    for i in range(40):
        n = int(rng.choice([128, 256, 512]))
        k = int(rng.choice([3, 10, 40]))
        snr = float(rng.choice([10.0, 20.0, 30.0]))
        b0 = int(rng.choice([4, 8, 16, 32, 64]))
        eps1 = float(rng.uniform(0.05, 0.9))
        eps2 = float(rng.uniform(0.2, 2.0))
        d1 = float(rng.uniform(0.005, 0.1))
        d2 = float(d1 + rng.uniform(0.01, 0.3))
        iters = [None, 1, 3, 6, 12, 25][int(rng.integers(0, 6))]
        mag_floor = float(rng.choice([1e-3, 0.05, 0.2, 0.6]))
        prune = float(rng.choice([0.0, 1e-3, 0.3]))
        loops = int(rng.choice([1, 2, 3, 8]))
        cases.append((i, n, k, snr, b0, eps1, eps2, d1, d2, iters, mag_floor, prune, loops))
    # edges: start bins below the minimum grid and above the image side, no
    # tuning iterations at all, a single loop, an image of pure noise
    for j, (n, k, snr, b0, iters, loops) in enumerate([
            (128, 5, 20.0, 1, None, 3), (128, 5, 20.0, 2, 4, 8), (128, 5, 20.0, 1024, None, 2),
            (256, 5, 20.0, 16, 0, 8), (256, 0, 20.0, 16, None, 8), (64, 2, 40.0, 64, None, 1)]):
        cases.append((len(cases), n, k, snr, b0, 0.5, 1.0, 0.02, 0.05, iters, 1e-3, 1e-3, loops))
    return cases


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: f"fuzz{c[0]}")
def test_atsfft_config_fuzz_vs_oracle(case):
    """Random tuner configurations (start bins, ratio thresholds, convergence
    band, iteration caps including 1, magnitude floors, prune levels, loop
    counts) on noisy images: every branch of update_bins, the cycle guard, the
    iteration cap and the vote-budget fallback (tuner.py:121-241) against the
    oracle — trajectory, state, support in dict order, values 1e-10."""
    i, n, k, snr, b0, eps1, eps2, d1, d2, iters, mag_floor, prune, loops = case
    img = P.sparse_image(n, k, 100 + i, snr_db=snr, dtype=np.complex128)
    cfg = P.TunerConfig(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, max_tuning_iters=iters,
                        mag_floor=mag_floor, prune_rel=prune)
    oc = O.TunerParams(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, max_iters=iters,
                       mag_floor=mag_floor, prune_rel=prune)
    try:
        (cs, vs), ostate = O.atsfft(img.x, oc, loops, 50 + i)
        oerr = None
    except O.OracleConfigError as e:
        oerr = e
    if oerr is not None:
        with pytest.raises(P.ConfigurationError):
            P.atsfft2d(img.x, cfg, loops, 50 + i, precision="fp64")
        return
    got, state = P.atsfft2d(img.x, cfg, loops, 50 + i, precision="fp64")
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    assert (state.converged, state.detected_k, state.b_estimate, state.vote_passes) == \
        (ostate["converged"], ostate["detected_k"], ostate["b_estimate"], ostate["vote_passes"])
    _fuzz_compare(got, O.as_dict((cs, vs)))


def _sfft_fuzz_cases():
    rng = np.random.default_rng(77)
    cases = []
    for i in range(40):
        n = int(rng.choice([64, 128, 256, 512]))
        k = int(rng.choice([1, 3, 10, 30]))
        snr = [None, 10.0, 30.0][int(rng.integers(0, 3))]
        loops = int(rng.choice([1, 2, 3, 5, 8, 11]))
        d_factor = int(rng.choice([1, 2, 4]))
        thr = int(rng.integers(1, loops + 1))
        b = int(rng.choice([b for b in (4, 8, 16, 32, 64, 128) if b <= n]))
        prune = float(rng.choice([0.0, 1e-3, 0.5]))
        cases.append((i, n, k, snr, loops, d_factor, thr, b, prune))
    # edges: every bin kept (d_factor * k = B^2), w = 1 (B = N), the smallest
    # grid, k = 0 (one kept bin, engine.py:116-118)
    for n, k, snr, loops, d_factor, thr, b in [
            (64, 8, 20.0, 3, 2, 2, 4), (128, 16, None, 5, 1, 3, 4), (64, 3, 20.0, 4, 2, 2, 64),
            (64, 1, None, 1, 1, 1, 4), (128, 0, 20.0, 3, 2, 2, 16)]:
        cases.append((len(cases), n, k, snr, loops, d_factor, thr, b, 1e-3))
    return cases


@pytest.mark.parametrize("case", _sfft_fuzz_cases(), ids=lambda c: f"sfuzz{c[0]}")
def test_sfft_config_fuzz_vs_oracle(case):
    """Random Algorithm 1 configurations (loop counts above and below 8, every
    vote threshold, kept-bin factors, bin counts from 4 to 128, prune levels;
    noiseless and noisy images) against the oracle: support in dict order and
    values 1e-10; configurations the reference rejects must be rejected."""
    i, n, k, snr, loops, d_factor, thr, b, prune = case
    img = (P.planted_image(n, k, 300 + i) if snr is None
           else P.sparse_image(n, k, 300 + i, snr_db=snr, dtype=np.complex128))
    kw = dict(loops=loops, d_factor=d_factor, vote_threshold=thr, b_bins=b, prune_rel=prune)
    try:
        oc = O.sfft_params(n, k, **kw)
    except O.OracleConfigError:
        with pytest.raises(P.ConfigurationError):
            P.sfft2d(img.x, P.SfftConfig(n=n, k=k, **kw), 70 + i, precision="fp64")
        return
    want = O.as_dict(O.sfft(img.x, oc, 70 + i))
    got = P.sfft2d(img.x, P.SfftConfig(n=n, k=k, **kw), 70 + i, precision="fp64")
    _fuzz_compare(got, want)


def _fold_fuzz_cases():
    rng = np.random.default_rng(909)
    cases = []
    for i in range(36):
        n = int(rng.choice([64, 128, 256, 512, 1024, 2048, 4096], p=[.1, .15, .2, .2, .15, .12, .08]))
        b = int(rng.choice([v for v in (4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096) if v <= n]))
        loops = int(rng.choice([1, 1, 2, 3, 8]))
        dt = [np.complex64, np.complex128][int(rng.integers(0, 2))]
        cases.append((i, n, b, loops, dt))
    return cases


@pytest.mark.parametrize("case", _fold_fuzz_cases(), ids=lambda c: f"fold{c[0]}-n{c[1]}-b{c[2]}-l{c[3]}")
def test_binned_spectrum_geometry_fuzz_vs_oracle(case):
    """Every fold geometry (k_fold / k_fold_ml / TMA ring / wide, partial-sum
    slices, single and multi-loop launches, whole-grid and four-step FFTs)
    over random (N, B, loops, input dtype) against the oracle's bucket
    spectrum (hashing.py:308-337), 1e-12."""
    i, n, b, loops, dt = case
    rng = np.random.default_rng(1000 + i)
    x = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(dt)
    win = P.build_flat_window(n, b, 1e-8, delta_pass=1e-3)
    perms = [P.draw_permutation(n, rng) for _ in range(loops)]
    got = P.binned_spectrum(x, perms if loops > 1 else perms[0], win, b).spectrum
    got = got if loops > 1 else got[None]
    ow = O.window(n, b, 1e-8, 1e-3)
    a = O.as_c128(x)
    for l, p in enumerate(perms):
        ref = O.bucket_spectrum(a, O.make_perm(n, p.sigma1, p.sigma2, p.tau1, p.tau2), ow, b)
        assert np.abs(got[l] - ref).max() <= 1e-12 * np.abs(ref).max(), (n, b, l)


@pytest.mark.parametrize("case", _fuzz_cases()[:24], ids=lambda c: f"dfuzz{c[0]}")
def test_detect_sparsity_fuzz_votes_vs_oracle(case):
    """The tuner's vote accumulation (tuner.py:165-179, 228-240) under the same
    random configurations: every voted coordinate and its tally (deferred
    shared-memory tallies, bitmap and list passes, the early tally, the
    over-budget fallback) must equal the oracle's, with the trajectory."""
    i, n, k, snr, b0, eps1, eps2, d1, d2, iters, mag_floor, prune, loops = case
    img = P.sparse_image(n, k, 100 + i, snr_db=snr, dtype=np.complex128)
    cfg = P.TunerConfig(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, max_tuning_iters=iters,
                        mag_floor=mag_floor)
    oc = O.TunerParams(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, max_iters=iters,
                       mag_floor=mag_floor)
    ostate, (ocoords, otal), _ = O.detect(O.as_c128(img.x), oc, np.random.default_rng(50 + i))
    state, (coords, tallies) = P.detect_sparsity(img.x, cfg, 50 + i)
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    assert state.vote_passes == ostate["vote_passes"]
    np.testing.assert_array_equal(coords, ocoords)
    np.testing.assert_array_equal(tallies, otal)


@pytest.mark.parametrize("case", _fuzz_cases()[:24], ids=lambda c: f"f32fuzz{c[0]}")
def test_atsfft_config_fuzz_fp32_vs_oracle(case):
    """The fp32 path under the same random configurations: support equal to
    the oracle's (a coefficient within 1e-4 of a selection boundary may fall
    on either side), values within 1e-4.  A count near-tie among noise bins
    can flip in fp32 and change the bin trajectory; such a case is compared
    only up to the first pass whose count differs, which must differ by less
    than 1e-4 relative (at least 1 bin)."""
    i, n, k, snr, b0, eps1, eps2, d1, d2, iters, mag_floor, prune, loops = case
    img = P.sparse_image(n, k, 100 + i, snr_db=snr, dtype=np.complex128)
    cfg = P.TunerConfig(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, max_tuning_iters=iters,
                        mag_floor=mag_floor, prune_rel=prune)
    oc = O.TunerParams(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, max_iters=iters,
                       mag_floor=mag_floor, prune_rel=prune)
    (cs, vs), ostate = O.atsfft(img.x, oc, loops, 50 + i)
    got, state = P.atsfft2d(img.x, cfg, loops, 50 + i, precision="fp32")
    gh = [(b, c) for b, c, _ in state.history]
    oh = [(b, c) for b, c, _ in ostate["history"]]
    if gh != oh:
        # first differing pass: same bin count, local-maximum counts within 1e-4
        t = next((j for j, (a, b) in enumerate(zip(gh, oh)) if a != b), min(len(gh), len(oh)))
        assert t < min(len(gh), len(oh)), (gh, oh)
        assert gh[t][0] == oh[t][0]
        assert abs(gh[t][1] - oh[t][1]) <= max(1.0, 1e-4 * oh[t][1]), (t, gh[t], oh[t])
        pytest.skip("an fp32 count near-tie changed the trajectory")
    _close_values(got, O.as_dict((cs, vs)), 1e-4)


def _large_fuzz_cases():
    rng = np.random.default_rng(4242)
    cases = []
    for i, n in enumerate([1024, 1024, 1024, 1024, 2048, 2048]):
        k = int(rng.choice([20, 100]))
        snr = float(rng.choice([15.0, 25.0]))
        b0 = int(rng.choice([8, 16, 64, 128]))
        eps1 = float(rng.uniform(0.2, 0.8))
        eps2 = float(rng.uniform(0.6, 1.5))
        d1 = float(rng.uniform(0.005, 0.04))
        d2 = float(d1 + rng.uniform(0.02, 0.1))
        mag_floor = float(rng.choice([1e-3, 0.02]))
        loops = int(rng.choice([3, 8]))
        cases.append((i, n, k, snr, b0, eps1, eps2, d1, d2, None, mag_floor, 1e-3, loops))
    return cases


@pytest.mark.parametrize("case", _large_fuzz_cases(), ids=lambda c: f"lfuzz{c[0]}-n{c[1]}")
def test_atsfft_large_config_fuzz_vs_oracle(case):
    """Random tuner configurations at N = 1024 and 2048: the speculative paired
    folds, the B = N/2 pass from the dense spectrum (k_pass_conv_band), the
    register-window local maxima at B >= 128, bitmap and list vote passes, the
    early tally and the fused tail — trajectory, state, support, order and
    values against the oracle."""
    i, n, k, snr, b0, eps1, eps2, d1, d2, iters, mag_floor, prune, loops = case
    img = P.sparse_image(n, k, 700 + i, snr_db=snr, dtype=np.complex64)
    cfg = P.TunerConfig(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, mag_floor=mag_floor,
                        prune_rel=prune)
    oc = O.TunerParams(b0=b0, eps1=eps1, eps2=eps2, delta1=d1, delta2=d2, mag_floor=mag_floor,
                       prune_rel=prune)
    (cs, vs), ostate = O.atsfft(img.x, oc, loops, 800 + i)
    got, state = P.atsfft2d(img.x, cfg, loops, 800 + i, precision="fp64")
    assert [(b, c) for b, c, _ in state.history] == [(b, c) for b, c, _ in ostate["history"]]
    assert (state.converged, state.detected_k, state.b_estimate, state.vote_passes) == \
        (ostate["converged"], ostate["detected_k"], ostate["b_estimate"], ostate["vote_passes"])
    _fuzz_compare(got, O.as_dict((cs, vs)))
