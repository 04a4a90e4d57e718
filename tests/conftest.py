"""Shared test helpers.

Markers: ``gpu`` — needs a CUDA device (B200) and the built native library;
``slow`` — long CPU oracle runs, only with SFFT2D_SLOW=1.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200) and libsfft2d_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case (SFFT2D_SLOW=1)")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("SFFT2D_SLOW") == "1":
        return
    skip = pytest.mark.skip(reason="slow oracle case; set SFFT2D_SLOW=1")
    for item in items:
        if "slow" in item.keywords:
            item.add_marker(skip)


def golden(name):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return dict(np.load(path, allow_pickle=False))


def golden_names(prefix):
    if not os.path.isdir(GOLDEN):
        return []
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.startswith(prefix) and f.endswith(".npz"))


def fixture_input(g):
    """The input image of a golden case: stored, or regenerated + digest-checked."""
    from paper_1908_02461_b200.signals import image_digest, sparse_image
    if "x" in g:
        return g["x"]
    if "gen_planted" in g:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        n, k, seed = (int(v) for v in g["gen_planted"])
        x = _planted(n, k, seed).astype(np.complex64)
    else:
        kw = {}
        if "gen_snr" in g:
            kw["snr_db"] = float(g["gen_snr"])
        if "gen_mag" in g:
            kw["magnitude"] = str(g["gen_mag"])
        if "gen_cluster" in g:
            kw["cluster_frac"] = float(g["gen_cluster"])
        x = sparse_image(int(g["gen_n"]), int(g["gen_k"]), int(g["gen_seed"]), **kw).x
    assert image_digest(x) == str(g["digest"]), "regenerated input does not match the fixture"
    return x


def _planted(n, k, seed):
    # generate_planted (signals.py:42-65) restated: distinct flat draws, phases, outer products
    rng = np.random.default_rng(seed)
    flat = rng.choice(n * n, size=k, replace=False)
    ii, jj = flat // n, flat % n
    coeffs = np.exp(1j * rng.uniform(0.0, 2.0 * np.pi, size=k))
    grid = np.arange(n)
    ei = np.exp(2j * np.pi * np.outer(grid, ii) / n)
    ej = np.exp(2j * np.pi * np.outer(jj, grid) / n)
    return (ei * coeffs) @ ej / (n * n)


def perms_from_rows(rows, n):
    from oracle.sfft_oracle import Perm
    return [Perm(n, *[int(v) for v in r[:4]], int(r[4]), int(r[5])) for r in rows]


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def assert_int_array(got, g, key):
    """Exact comparison with a fixture array stored verbatim or as count + sha256."""
    import hashlib
    got = np.ascontiguousarray(np.asarray(got, dtype=np.int64))
    if key in g:
        np.testing.assert_array_equal(got, g[key])
        return
    assert got.size == int(g[key + "_n"]), (got.size, int(g[key + "_n"]))
    np.testing.assert_array_equal(got[: g[key + "_head"].size], g[key + "_head"])
    assert int(got.sum()) == int(g[key + "_sum"])
    assert hashlib.sha256(got.tobytes()).hexdigest() == str(g[key + "_sha"])
