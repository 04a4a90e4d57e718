"""torch.library custom ops over the C ABI (paper_1908_02461_b200.ops): they are
registered, their fake kernels give the right shapes (CPU), and on the GPU
they equal the Python API and trace under torch.compile."""

import numpy as np
import pytest
import torch

import paper_1908_02461_b200 as P
from paper_1908_02461_b200 import ops  # noqa: F401  (registers torch.ops.sfft2d_b200)
from oracle import sfft_oracle as O

gpu = pytest.mark.gpu
OPS = ["binned_spectrum", "bucket_fft2d", "top_bins", "local_maxima", "sfft", "atsfft"]


def test_ops_registered():
    for name in OPS:
        assert hasattr(torch.ops.sfft2d_b200, name), name


def test_fake_kernels_shapes():
    from torch._subclasses.fake_tensor import FakeTensorMode
    from torch.fx.experimental.symbolic_shapes import ShapeEnv
    with FakeTensorMode(shape_env=ShapeEnv()):
        x = torch.empty(256, 256, dtype=torch.complex64)
        perms = torch.empty(3, 6, dtype=torch.int64)
        g = torch.ops.sfft2d_b200.binned_spectrum(x, perms, 64, 1e-3, 1e-8, False)
        assert tuple(g.shape) == (3, 64, 64) and g.dtype == torch.complex64
        f = torch.ops.sfft2d_b200.bucket_fft2d(g, 256, True)
        assert tuple(f.shape) == (3, 64, 64) and f.dtype == torch.complex128
        t = torch.ops.sfft2d_b200.top_bins(g, 20, False)
        assert tuple(t.shape) == (3, 20) and t.dtype == torch.int32
        c = torch.ops.sfft2d_b200.local_maxima(g[0], 1e-3, False)
        assert c.dim() == 2 and c.shape[1] == 2 and c.dtype == torch.int64
        ij, v = torch.ops.sfft2d_b200.atsfft(x, 11, 8, 16, 0.5, 1.0, 0.02, 0.05, -1, 1e-3, 1e-3,
                                             1e-8, 1e-6, 1e-3, True)
        assert ij.shape[1] == 2 and v.dtype == torch.complex128 and v.shape[0] == ij.shape[0]


@gpu
def test_ops_equal_python_api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    img = P.sparse_image(256, 8, 4, snr_db=25.0)
    x = torch.from_numpy(img.x).cuda()
    p = [P.draw_permutation(256, np.random.default_rng(s)) for s in (1, 2)]
    win = P.build_flat_window(256, 64, 1e-8, delta_pass=1e-3)
    g = torch.ops.sfft2d_b200.binned_spectrum(x, ops.perms_tensor(p), 64, 1e-3, 1e-8, True)
    ref = P.binned_spectrum(x, p, win, 64).spectrum
    assert torch.equal(g, ref)
    t = torch.ops.sfft2d_b200.top_bins(g, 16, True).cpu().numpy()
    for s in range(2):
        np.testing.assert_array_equal(t[s], np.sort(O.top_bins(g[s].cpu().numpy(), 16)))
    c = torch.ops.sfft2d_b200.local_maxima(g[0], 1e-3, True).cpu().numpy()
    np.testing.assert_array_equal(c, P.count_local_maxima(g[0], 1e-3)[1])
    grid = torch.randn(2, 64, 64, dtype=torch.complex128, device="cuda")
    f = torch.ops.sfft2d_b200.bucket_fft2d(grid, 256, True)
    torch.testing.assert_close(f, torch.fft.fft2(grid), rtol=1e-12, atol=1e-10)
    ij, v = torch.ops.sfft2d_b200.atsfft(x, 11, 8, 16, 0.5, 1.0, 0.02, 0.05, -1, 1e-3, 1e-3, 1e-8,
                                         1e-6, 1e-3, True)
    (ij2, v2), _ = P.atsfft2d_arrays(x, P.TunerConfig(), 8, 11)
    np.testing.assert_array_equal(ij.cpu().numpy(), ij2)
    np.testing.assert_array_equal(v.cpu().numpy(), v2)
    sig = P.planted_image(256, 6, 3)
    xs = torch.from_numpy(sig.x).cuda()
    ij3, v3 = torch.ops.sfft2d_b200.sfft(xs, 2, 6, 8, 2, 0, 0, 1e-3, 1e-8, 1e-6, 1e-3, True)
    want = P.sfft2d(sig.x, P.SfftConfig(n=256, k=6), 2)
    got = {(int(i), int(j)): complex(z) for (i, j), z in zip(ij3.tolist(), v3.tolist())}
    assert got == want


@gpu
def test_ops_trace_under_compile():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    img = P.sparse_image(256, 8, 4, snr_db=25.0)
    x = torch.from_numpy(img.x).cuda()
    perms = ops.perms_tensor([P.draw_permutation(256, np.random.default_rng(3))])

    def f(x):
        g = torch.ops.sfft2d_b200.binned_spectrum(x, perms, 64, 1e-3, 1e-8, True)
        return torch.ops.sfft2d_b200.top_bins(g, 8, True)

    eager = f(x)
    compiled = torch.compile(f, fullgraph=True)(x)
    assert torch.equal(eager, compiled)
