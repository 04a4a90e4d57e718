"""Host-side split of one c3 atsfft2d_arrays call: total wall vs the native
call (ctx.last_call_us), plus a cProfile of the Python layer.
python tools/py_split.py [fp32|fp64]"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
img = P.sparse_image(4096, 100, 7, snr_db=20.0)
x = torch.from_numpy(img.x).cuda()
cfg = P.TunerConfig()
ctx = _native.context(0)
for _ in range(5):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision=prec)
torch.cuda.synchronize()
tot, nat = [], []
for _ in range(50):
    t0 = time.perf_counter()
    P.atsfft2d_arrays(x, cfg, 8, 11, precision=prec)
    tot.append((time.perf_counter() - t0) * 1e6)
    nat.append(ctx.last_call_us)
print(f"total {np.median(tot):.1f} us, native call {np.median(nat):.1f} us, python {np.median(tot) - np.median(nat):.1f} us")
t0 = time.perf_counter()
for _ in range(200):
    np.random.default_rng(11)
print(f"default_rng(11): {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(100):
    P.atsfft2d_arrays(x, cfg, 8, 11, precision=prec)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
