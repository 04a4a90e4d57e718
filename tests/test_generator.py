"""Device workload generator: the Philox restatement
is pinned to the published known-answer vectors on CPU; the device image
(`sfft2d_generate` through `signals.device_sparse_image`) is compared with
that restatement on the GPU."""

import numpy as np
import pytest

from oracle import generator_oracle as G
from paper_1908_02461_b200 import signals as S

# Random123 known-answer vectors for philox4x32_10 (ctr, key -> out)
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KAT)
def test_philox_known_answers(ctr, key, want):
    got = G.philox4x32_10(np.array([ctr], dtype=np.uint64), key)[0]
    assert tuple(int(v) for v in got) == want


def test_noise_is_standard_normal():
    n1, n2 = G.noise(1 << 18, 12345)
    for v in (n1, n2):
        assert abs(v.mean()) < 0.01 and abs(v.var() - 1.0) < 0.01
    assert abs(np.corrcoef(n1, n2)[0, 1]) < 0.01


def test_clean_part_matches_host_generator():
    # same seed -> same coefficients as sparse_image; noiseless images agree
    host = S.sparse_image(256, 12, 9, magnitude="loguniform", cluster_frac=0.25, cluster_side=16,
                          dtype=np.complex128)
    rng = np.random.default_rng(9)
    rows, cols, coeffs = S._draw_spectrum(rng, 256, 12, "loguniform", (0.1, 10.0), 0.25, 16)
    np.testing.assert_array_equal(rows, host.rows)
    np.testing.assert_array_equal(cols, host.cols)
    np.testing.assert_array_equal(coeffs, host.coeffs)
    x = G.device_image(256, rows, cols, coeffs, 0.0, 0, dtype=np.complex128)
    np.testing.assert_allclose(x, host.x, rtol=0, atol=1e-15)


def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.gpu
@pytest.mark.parametrize("n,k,snr,dtype", [(256, 10, 20.0, np.complex128), (1024, 50, 30.0, np.complex64),
                                           (1024, 150, 25.0, np.complex128), (4096, 100, 20.0, np.complex64),
                                           (512, 0, 10.0, np.complex64), (128, 5, None, np.complex64)])
def test_device_image_matches_restatement(n, k, snr, dtype):
    _need_gpu()
    img = S.device_sparse_image(n, k, 7, snr_db=snr, magnitude="loguniform", dtype=dtype)
    got = img.x.cpu().numpy()
    want = G.device_image(n, img.rows, img.cols, img.coeffs, img.noise_sd, img.noise_seed,
                          dtype=np.complex128)
    scale = np.abs(want).max() if k or snr else 1.0
    tol = 1e-12 if dtype == np.complex128 else 2e-6
    assert np.abs(got - want).max() <= tol * max(scale, 1e-300)
    if snr is not None and k:
        clean = G.device_image(n, img.rows, img.cols, img.coeffs, 0.0, 0, dtype=np.complex128)
        meas = 10 * np.log10(np.mean(np.abs(clean) ** 2) / np.mean(np.abs(want - clean) ** 2))
        assert abs(meas - snr) < 0.1


@pytest.mark.gpu
def test_device_image_deterministic_and_errors():
    _need_gpu()
    import torch
    a = S.device_sparse_image(512, 20, 3, snr_db=25.0).x
    b = S.device_sparse_image(512, 20, 3, snr_db=25.0).x
    assert torch.equal(a, b)
    out = torch.empty((512, 512), dtype=torch.complex64, device="cuda")
    c = S.device_sparse_image(512, 20, 3, snr_db=25.0, out=out)
    assert c.x.data_ptr() == out.data_ptr() and torch.equal(out, a)
    with pytest.raises(ValueError):
        S.device_sparse_image(500, 3, 1)
    with pytest.raises(ValueError):
        S.device_sparse_image(64, 3, 1, out=torch.empty((32, 32), dtype=torch.complex64, device="cuda"))


@pytest.mark.gpu
def test_device_image_transform_recovers_truth():
    # a device-generated c2-style image goes through atsfft2d and recovers the
    # planted support (30 dB, k = 50)
    _need_gpu()
    import paper_1908_02461_b200 as P
    img = S.device_sparse_image(1024, 50, 7, snr_db=30.0)
    out, state = P.atsfft2d(img.x, P.TunerConfig(), 8, 11, precision="fp32")
    assert set(img.truth) <= set(out)
