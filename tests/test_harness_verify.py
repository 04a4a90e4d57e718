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


# ---------------------------------------------------------------- harness (§8(f) row 1)
REF_CSV = os.path.join(os.path.dirname(__file__), "golden", "ref_harness_tiny.csv")
TINY = dict(sizes=(64, 128), sparsities=(4,), trials=3, seed=11)


def test_planted_signal_is_the_references_image():
    from tests.conftest import golden
    g = golden("c1_sfft")          # x = reference generate_planted(256, 10, 1)
    sig = harness.planted_signal(256, 10, 1)
    assert sig.x.dtype == np.complex128
    np.testing.assert_array_equal(sig.x, g["x"])


def test_harness_spec_validation():
    with pytest.raises(ValueError):
        harness.ExperimentSpec(algorithms=("fftw",))
    with pytest.raises(ValueError):
        harness.ExperimentSpec(sizes=(12,))
    with pytest.raises(ValueError):
        harness.ExperimentSpec(trials=0)
    with pytest.raises(ValueError):
        harness.ExperimentSpec(precision="fp16")


def test_harness_csv_summary_tables_with_reference_rows(tmp_path):
    ref_rows = harness.read_rows_csv(REF_CSV)
    assert len(ref_rows) == 18 and {r.algorithm for r in ref_rows} == {"dense", "sfft", "atsfft"}
    # synthetic GPU rows, 100x faster than the reference's cells
    gpu = [harness.ResultRow("gpu-" + r.algorithm if r.algorithm != "dense" else "cufft-dense",
                             r.n, r.k, r.trial, r.wall_time_seconds / 100, r.error_metric,
                             r.detected_k, r.converged, r.b_final, r.status, 0.0)
           for r in ref_rows]
    path = tmp_path / "gpu.csv"
    harness.write_rows_csv(gpu, path)
    back = harness.read_rows_csv(path)
    assert [(r.algorithm, r.n, r.trial, r.error_metric, r.detected_k, r.converged, r.b_final)
            for r in back] == [(r.algorithm, r.n, r.trial, r.error_metric, r.detected_k,
                                r.converged, r.b_final) for r in gpu]
    summary = harness.summarize(back + ref_rows)
    assert summary.algorithms() == ["gpu-sfft", "gpu-atsfft", "cufft-dense", "dense", "sfft",
                                    "atsfft"]
    for n in (64, 128):
        assert summary.speedup("gpu-sfft", "sfft", n, 4) == pytest.approx(100.0)
        assert summary.speedup("gpu-atsfft", "atsfft", n, 4) == pytest.approx(100.0)
    tables = harness.summary_tables(summary)
    text = harness.render_tables_text(tables)
    assert "gpu-atsfft/atsfft speedup" in text and "100.00x" in text
    assert "gpu-atsfft detection rate" in text
    csv_text = harness.render_tables_csv(tables)
    assert csv_text.startswith("# runtime and speedup, k=4\nmetric,n=64,n=128\n")
    spec = harness.ExperimentSpec(**TINY)
    harness.write_sidecar(spec, tmp_path / "gpu.json")
    side = __import__("json").load(open(tmp_path / "gpu.json"))
    assert side["spec"]["sizes"] == [64, 128] and "cpu_model" in side["environment"]


@gpu
def test_harness_reproduces_reference_rows():
    """Same grid as the reference's own harness run (tests/golden/ref_harness_tiny.csv):
    every cell sees the same image and permutations, so the error, detected k,
    convergence and final B columns agree (fp64)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ref = {(r.algorithm, r.n, r.k, r.trial): r for r in harness.read_rows_csv(REF_CSV)}
    rows = harness.run_experiment(harness.ExperimentSpec(**TINY))
    assert len(rows) == 18
    name = {"gpu-sfft": "sfft", "gpu-atsfft": "atsfft", "cufft-dense": "dense"}
    for r in rows:
        want = ref[(name[r.algorithm], r.n, r.k, r.trial)]
        assert r.status == want.status == "ok"
        assert abs(r.error_metric - want.error_metric) <= 1e-9, (r, want)
        assert (r.detected_k, r.converged, r.b_final) == (want.detected_k, want.converged,
                                                          want.b_final), (r, want)
    summary = harness.summarize(rows + list(ref.values()))
    assert summary.speedup("gpu-atsfft", "atsfft", 128, 4) is not None
