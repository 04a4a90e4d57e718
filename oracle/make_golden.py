"""Generate golden fixtures by running the REAL reference (dev container only).

    python oracle/make_golden.py [case ...]        # default: every case

Imports ``sfft2d`` read-only from ``/root/reference/pkg/src`` and writes
``tests/golden/<case>.npz``.  Inputs come from the package's seeded workload
generator (``paper_1908_02461_b200.signals``); large inputs are NOT stored —
the fixture keeps the seed/parameters and a sha256 of the input bytes so a test
can regenerate and verify it.  Small inputs are stored verbatim.

This script is test infrastructure: it never runs on the GPU box (the
reference tree does not exist there) and nothing in the product imports it.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import sfft2d as ref  # noqa: E402
from sfft2d import engine as ref_engine  # noqa: E402
from sfft2d import hashing as ref_hashing  # noqa: E402

from paper_1908_02461_b200.signals import image_digest, sparse_image  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


BIG = 50_000


def digest_array(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def shrink(arrays: dict) -> dict:
    """Large vote lists are pinned by count + sha256 (+ a head sample), keeping
    fixtures small; tests compare digests of the full arrays."""
    out = dict(arrays)
    for key in ("vote_keys", "vote_tallies", "cand_keys"):
        if key in out and np.asarray(out[key]).size > BIG:
            a = np.asarray(out.pop(key), dtype=np.int64)
            out[key + "_sha"] = np.array(digest_array(a))
            out[key + "_n"] = np.array(a.size)
            out[key + "_sum"] = np.array(int(a.sum()))
            out[key + "_head"] = a[:2000]
    return out


def _save(name, **arrays):
    arrays = shrink(arrays)
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


def _dict_arrays(d: dict):
    keys = list(d)
    coords = np.array(keys, dtype=np.int64).reshape(-1, 2)
    vals = np.array([d[k] for k in keys], dtype=np.complex128)
    return coords, vals


def _hist_arrays(state):
    h = np.array([(b, c, np.nan if r is None else r) for b, c, r in state.history],
                 dtype=np.float64).reshape(-1, 3)
    none = np.array([r is None for _, _, r in state.history], dtype=bool)
    return h, none


def _perm_row(p):
    return [p.sigma1, p.sigma2, p.tau1, p.tau2, p.sigma1_inv, p.sigma2_inv]


# ---------------------------------------------------------------- cases
def case_windows():
    rows, spaces, freqs = [], [], []
    for (n, dstop, dpass) in [(16, 1e-8, 1e-6), (64, 1e-8, 1e-6), (256, 1e-8, 1e-6),
                              (64, 1e-8, 1e-3), (256, 1e-8, 1e-3), (1024, 1e-8, 1e-3),
                              (4096, 1e-8, 1e-3), (512, 1e-4, 1e-2)]:
        b = 4
        while b <= n:
            w = ref_hashing.build_flat_window(n, b, dstop, delta_pass=dpass)
            rows.append([n, b, dstop, dpass, w.support_w, w.half_support, w.pass_halfwidth])
            spaces.append(w.space_1d)
            freqs.append(w.freq_1d)
            b *= 2
    meta = np.array(rows, dtype=np.float64)
    _save("windows", meta=meta, space=np.concatenate(spaces), freq=np.concatenate(freqs))


def case_windows_16384():
    rows = []
    b = 4
    while b <= 16384:
        w = ref_hashing.build_flat_window(16384, b, 1e-8, delta_pass=1e-3)
        rows.append([16384, b, w.support_w, w.half_support, float(w.space_1d.sum()),
                     float(np.abs(w.space_1d).max()), float(w.freq_1d[1])])
        b *= 2
    _save("windows_16384", meta=np.array(rows, dtype=np.float64))


def case_binned():
    out = {}
    cases = [(16, 4, 1e-8, 1e-6), (64, 8, 1e-8, 1e-3), (256, 16, 1e-8, 1e-3),
             (256, 64, 1e-8, 1e-3), (512, 8, 1e-8, 1e-3), (1024, 32, 1e-8, 1e-3),
             (1024, 128, 1e-8, 1e-3), (256, 256, 1e-8, 1e-3), (128, 4, 1e-8, 1e-3)]
    for idx, (n, b, dstop, dpass) in enumerate(cases):
        # per-case stream: x (complex64) then the permutation; large x are regenerated
        rng = np.random.default_rng(1000 + idx)
        x = (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n))).astype(np.complex64)
        win = ref_hashing.build_flat_window(n, b, dstop, delta_pass=dpass)
        p = ref_hashing.draw_permutation(n, rng)
        spec = ref_hashing.binned_spectrum(x, p, win, b).spectrum
        if n <= 256:
            out[f"x{idx}"] = x
        out[f"spec{idx}"] = spec
        out[f"perm{idx}"] = np.array(_perm_row(p), dtype=np.int64)
        out[f"cfg{idx}"] = np.array([n, b, dstop, dpass, 1000 + idx], dtype=np.float64)
    _save("binned", ncases=np.array(len(cases)), **out)


def case_localmax():
    from sfft2d.tuner import count_local_maxima
    rng = np.random.default_rng(5)
    out = {}
    grids = [rng.normal(size=(16, 16)) + 1j * rng.normal(size=(16, 16)),
             rng.normal(size=(64, 64)) + 1j * rng.normal(size=(64, 64)),
             np.abs(rng.normal(size=(128, 128))).round(1).astype(np.complex128)]
    z = np.zeros((8, 8), complex)
    z[2, 2] = z[2, 3] = 1.0
    grids.append(z)
    g = np.zeros((8, 8), complex)
    g[1, 1] = 10.0
    g[6, 6] = 5.0
    g[4, 2] = 1e-4
    grids.append(g)
    grids.append(np.zeros((8, 8), complex))
    # non-power-of-two sides: the reference accepts any square grid >= 4x4
    for side in (5, 12, 100):
        grids.append(rng.normal(size=(side, side)) + 1j * rng.normal(size=(side, side)))
    grids.append(np.abs(rng.normal(size=(6, 6))).round(1).astype(np.complex128))
    for i, gr in enumerate(grids):
        cnt, coords = count_local_maxima(gr, 1e-3)
        out[f"grid{i}"] = gr
        out[f"count{i}"] = np.array(cnt)
        out[f"coords{i}"] = coords.astype(np.int64)
    _save("localmax", ngrids=np.array(len(grids)), **out)


def _sfft_case(name, x, n, k, seed, store_x, extra=None, **cfgkw):
    cfg = ref.SfftConfig(n=n, k=k, **cfgkw)
    t0 = time.perf_counter()
    out = ref.sfft2d(x, cfg, seed)
    dt = time.perf_counter() - t0
    # intermediate: location keys and voted coords, replayed with the same streams
    gen = np.random.default_rng(seed)
    kids = [np.random.default_rng(int(gen.integers(2**63))) for _ in range(2 * cfg.loops)]
    win = cfg.window()
    cand = []
    perms = []
    for i in range(cfg.loops):
        p, c = ref_engine.seek_location_once(np.asarray(x, np.complex128), cfg, win, kids[i])
        cand.append(c)
        perms.append(_perm_row(p))
    voted = ref_engine.vote_and_select(cand, cfg)
    for i in range(cfg.loops):
        perms.append(_perm_row(ref_hashing.draw_permutation(n, kids[cfg.loops + i])))
    coords, vals = _dict_arrays(out)
    arrays = dict(coords=coords, vals=vals, voted=voted.astype(np.int64),
                  perms=np.array(perms, dtype=np.int64),
                  cand_sizes=np.array([c.shape[0] for c in cand]),
                  cand_keys=np.concatenate([c[:, 0] * n + c[:, 1] for c in cand]),
                  cfg=np.array([n, k, cfg.loops, cfg.b_bins, cfg.vote_threshold, seed]),
                  ref_seconds=np.array(dt))
    if store_x:
        arrays["x"] = x
    if extra:
        arrays.update(extra)
    _save(name, **arrays)


def _ats_case(name, x, est_loops, seed, store_x, extra=None, **tkw):
    cfg = ref.TunerConfig(**tkw)
    t0 = time.perf_counter()
    out, state = ref.atsfft2d(x, cfg, est_loops, seed)
    dt = time.perf_counter() - t0
    # replay detection alone for the votes (same stream start); skipped for
    # the 16384^2 case (another ~20 min) — its votes are pinned by count only
    if np.asarray(x).shape[0] <= 4096:
        st2, (vc, vt) = ref.detect_sparsity(x, cfg, np.random.default_rng(seed))
        assert st2.history == state.history
    else:
        vc, vt = np.empty((0, 2), np.int64), np.empty(0, np.int64)
    coords, vals = _dict_arrays(out)
    hist, none = _hist_arrays(state)
    n = np.asarray(x).shape[0]
    arrays = dict(coords=coords, vals=vals, hist=hist, hist_none=none,
                  state=np.array([state.converged, state.detected_k, state.b_detect,
                                  state.b_estimate, state.vote_passes], dtype=np.int64),
                  vote_keys=(vc[:, 0] * n + vc[:, 1]).astype(np.int64),
                  vote_tallies=vt.astype(np.int64), est_loops=np.array(est_loops),
                  seed=np.array(seed), ref_seconds=np.array(dt),
                  tuner=np.array([cfg.b0, cfg.eps1, cfg.eps2, cfg.delta1, cfg.delta2,
                                  -1 if cfg.max_tuning_iters is None else cfg.max_tuning_iters,
                                  cfg.mag_floor], dtype=np.float64))
    if store_x:
        arrays["x"] = np.asarray(x)
    if extra:
        arrays.update(extra)
    _save(name, **arrays)
    print(f"  {name}: {dt:.2f}s hist={state.history[:3]}... det_k={state.detected_k} "
          f"out={len(out)}", flush=True)


def _gen_meta(img, **kw):
    meta = dict(gen_n=np.array(img.n), gen_k=np.array(img.k), gen_seed=np.array(img.seed),
                digest=np.array(image_digest(img.x)), truth_rows=img.rows, truth_cols=img.cols,
                truth_coeffs=img.coeffs)
    for key, v in kw.items():
        meta[f"gen_{key}"] = np.array(v)
    return meta


def case_c1():
    sig = ref.generate_planted(256, 10, 1)
    _sfft_case("c1_sfft", sig.x, 256, 10, 2, True)


def case_sfft_small():
    sig = ref.generate_planted(64, 4, 9)
    _sfft_case("sfft_n64_k4", sig.x, 64, 4, 10, True)
    sig = ref.generate_planted(128, 4, 77)
    _sfft_case("sfft_n128_k4", sig.x, 128, 4, 42, True)
    sig = ref.generate_planted(2048, 2, 44)
    _sfft_case("sfft_n2048_k2_b64", sig.x.astype(np.complex64), 2048, 2, 45, False,
               extra=dict(gen_planted=np.array([2048, 2, 44]),
                          digest=np.array(image_digest(sig.x.astype(np.complex64)))),
               b_bins=64)
    # degenerate full-size bins with loops=1 and no pruning
    rng = np.random.default_rng(3)
    x = rng.normal(size=(16, 16)) + 1j * rng.normal(size=(16, 16))
    _sfft_case("sfft_n16_bn", x, 16, 2, 3, True, loops=1, b_bins=16, prune_rel=0.0)
    _sfft_case("sfft_zero", np.zeros((64, 64)), 64, 2, 1, True)
    img = sparse_image(256, 12, 21, snr_db=20.0, magnitude="loguniform")
    _sfft_case("sfft_n256_noisy", img.x, 256, 12, 22, True, extra=_gen_meta(img, snr=20.0))


def case_ats_small():
    sig = ref.generate_planted(256, 8, 300)
    _ats_case("ats_n256_k8", sig.x, 8, 400, True)
    sig = ref.generate_planted(64, 1, 11)
    _ats_case("ats_n64_k1_b8", sig.x, 8, 12, True, b0=8)
    n = 64
    xhat = np.zeros((n, n), complex)
    xhat[0, 0] = 1.0
    _ats_case("ats_dc", ref.ifft2d(xhat), 8, 5, True, b0=8)
    _ats_case("ats_zero", np.zeros((64, 64)), 4, 6, True)
    sig = ref.generate_planted(64, 3, 900)
    _ats_case("ats_noconv", sig.x, 4, 901, True, max_tuning_iters=2)
    img = sparse_image(256, 10, 3, snr_db=20.0)
    _ats_case("ats_n256_20db", img.x, 8, 4, True, extra=_gen_meta(img, snr=20.0))
    img = sparse_image(512, 20, 5, snr_db=25.0, magnitude="loguniform")
    _ats_case("ats_n512_25db", img.x, 8, 6, False, extra=_gen_meta(img, snr=25.0, mag="loguniform"))
    img = sparse_image(128, 6, 8, snr_db=15.0)
    _ats_case("ats_n128_15db", img.x, 6, 9, True, extra=_gen_meta(img, snr=15.0))


def case_c2():
    img = sparse_image(1024, 50, 7, snr_db=30.0)
    _ats_case("c2_ats", img.x, 8, 11, False, extra=_gen_meta(img, snr=30.0))


def case_c2_sfft():
    img = sparse_image(1024, 50, 7, snr_db=30.0)
    _sfft_case("c2_sfft", img.x, 1024, 50, 12, False, extra=_gen_meta(img, snr=30.0))


def case_c3():
    img = sparse_image(4096, 100, 7, snr_db=20.0)
    _ats_case("c3_ats", img.x, 8, 11, False, extra=_gen_meta(img, snr=20.0))


def case_c3_sfft():
    img = sparse_image(4096, 100, 7, snr_db=20.0)
    _sfft_case("c3_sfft", img.x, 4096, 100, 12, False, extra=_gen_meta(img, snr=20.0))


def case_c3_clean():
    img = sparse_image(4096, 100, 7, snr_db=None)
    _ats_case("c3_ats_clean", img.x, 8, 11, False, extra=_gen_meta(img))


def case_c4():
    img = sparse_image(1024, 20, 1, snr_db=25.0, magnitude="loguniform")
    _ats_case("c4_k20", img.x, 8, 101, False, extra=_gen_meta(img, snr=25.0, mag="loguniform"))
    img = sparse_image(1024, 200, 2, snr_db=25.0, magnitude="loguniform")
    _ats_case("c4_k200", img.x, 8, 102, False, extra=_gen_meta(img, snr=25.0, mag="loguniform"))


def c4_bench_image(i: int):
    """bench.py's c4 image i (same definition as bench.c4_image): seed 100000 + i,
    k ~ U[20, 200] from that seed, log-uniform magnitudes, 25 dB."""
    seed = 100_000 + i
    k = int(np.random.default_rng(seed).integers(20, 201))
    return sparse_image(1024, k, seed, snr_db=25.0, magnitude="loguniform")


def case_c4_batch():
    # the first 12 images of the bench's c4 batch (rng seed 1 + i, as in the
    # bench leg), so the batched leg carries a parity spot-check
    for i in range(12):
        img = c4_bench_image(i)
        _ats_case(f"c4b_{i:02d}", img.x, 8, 1 + i, False,
                  extra=_gen_meta(img, snr=25.0, mag="loguniform", index=i))


def _c5_sweep(k, seed):
    img = sparse_image(16384, k, seed, snr_db=15.0, cluster_frac=0.2, cluster_side=64)
    x = img.x
    meta = _gen_meta(img, snr=15.0, cluster=0.2)
    del img
    _ats_case(f"c5_ats_k{k}", x, 8, seed + 1, False, extra=meta)


def case_c5_k256():
    _c5_sweep(256, 5)


def case_c5_k1024():
    _c5_sweep(1024, 5)


def case_c5_k4096():
    _c5_sweep(4096, 5)


def case_c5():
    # 16384^2 complex64, k=64, 20% in the wrap-around DC 64x64 block, 15 dB
    img = sparse_image(16384, 64, 5, snr_db=15.0, cluster_frac=0.2, cluster_side=64)
    x = img.x
    meta = _gen_meta(img, snr=15.0, cluster=0.2)
    del img
    _ats_case("c5_ats_k64", x, 8, 6, False, extra=meta)


def case_harness():
    """The reference harness's own rows for a tiny grid (bench.py:142-187),
    as its CSV: the GPU harness must reproduce the error / detection columns
    cell by cell (same signal and algorithm seeds)."""
    from sfft2d import bench as ref_bench
    spec = ref_bench.ExperimentSpec(algorithms=("dense", "sfft", "atsfft"), sizes=(64, 128),
                                    sparsities=(4,), trials=3, seed=11)
    rows = ref_bench.run_experiment(spec)
    ref_bench.write_rows_csv(rows, os.path.join(OUT, "ref_harness_tiny.csv"))


CASES = {name[5:]: fn for name, fn in globals().items() if name.startswith("case_")}

if __name__ == "__main__":
    todo = sys.argv[1:] or list(CASES)
    for name in todo:
        t0 = time.perf_counter()
        CASES[name]()
        print(f"[{name}] {time.perf_counter() - t0:.1f}s", flush=True)
