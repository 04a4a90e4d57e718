"""SF2D exchange format (host), harness algorithm names
and the verification suite on the GPU path."""

import os
import tempfile

import numpy as np
import pytest
import torch

import paper_1908_02461_b200 as P
from paper_1908_02461_b200 import harness, verify
from paper_1908_02461_b200.signals import load_signal, save_signal

gpu = pytest.mark.gpu


def test_sf2d_round_trip_and_layout():
    sig = P.sparse_image(32, 5, 9, snr_db=10.0, dtype=np.complex128)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "s.sf2d")
        save_signal(sig, path)
        raw = open(path, "rb").read()
        assert raw[:4] == b"SF2D" and len(raw) == 20 + 32 * 32 * 16
        assert int.from_bytes(raw[4:8], "little") == 32 and int.from_bytes(raw[8:12], "little") == 5
        assert int.from_bytes(raw[12:20], "little") == 9
        # payload: row-major little-endian float64 (re, im)
        first = np.frombuffer(raw[20:36], dtype="<f8")
        assert first[0] == sig.x[0, 0].real and first[1] == sig.x[0, 0].imag
        back = load_signal(path)
        assert (back.n, back.k, back.seed) == (32, 5, 9)
        np.testing.assert_array_equal(back.x, sig.x)
        open(path, "r+b").write(b"XXXX")
        with pytest.raises(ValueError):
            load_signal(path)


def test_harness_names():
    assert harness.ALGORITHMS == ("gpu-sfft", "gpu-atsfft", "cufft-dense")
    with pytest.raises(ValueError):
        harness.run_one("nope", P.planted_image(16, 1, 0))


@gpu
def test_harness_runs_each_algorithm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sig = P.planted_image(64, 4, 101)
    for algo in harness.ALGORITHMS:
        elapsed, err, dk, conv, b = harness.run_one(algo, sig, rng=202)
        assert elapsed > 0 and err <= 1e-6, (algo, err)


@gpu
def test_verify_suite_passes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lines = []
    assert verify.run_checks(out=lines.append), lines
    assert len(lines) == 10 and all(l.startswith("PASS") for l in lines)
