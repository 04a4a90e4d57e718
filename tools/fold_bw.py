"""Streaming-read calibration vs the fold kernel (binned_spectrum, one loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402

n = 4096
img = P.sparse_image(n, 100, 7, snr_db=20.0)
x = torch.from_numpy(img.x).cuda()
xf = torch.view_as_real(x).reshape(-1)
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


t = timeit(lambda: xf.sum())
print(f"torch sum of 134 MB: {t:.1f} us -> {134.2e6 / t / 1e3:.0f} GB/s")
t = timeit(lambda: x.clone())
print(f"torch clone 134 MB: {t:.1f} us -> {2 * 134.2e6 / t / 1e3:.0f} GB/s (r+w)")
rng = np.random.default_rng(1)
ctx = _native.context()
for b in (128, 256, 512, 1024, 2048):
    win = P.build_flat_window(n, b, 1e-8, delta_pass=1e-3)
    p = P.draw_permutation(n, rng)
    t = timeit(lambda: P.binned_spectrum(x, p, win, b, precision="fp32"))
    ctx.set_profiling(True)
    P.binned_spectrum(x, p, win, b, precision="fp32")
    rep = ctx.profile_report()
    ctx.set_profiling(False)
    ks = {k: v[1] * 1e3 for k, v in rep.items()}
    print(f"B={b:5d}: binned_spectrum {t:6.1f} us  " + "  ".join(f"{k}={v:.1f}" for k, v in ks.items()))
