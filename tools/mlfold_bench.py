"""k_fold_ml (SFFT multi-loop fold) time per launch: python tools/mlfold_bench.py [fp32|fp64]
Eight permutations folded from one read of the c3 image at B = 128 (the c3 known-k SFFT
location fold), per-launch CUDA-event times from the library's profiler, L2 flushed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
n = 4096
x = torch.from_numpy(P.sparse_image(n, 100, 7, snr_db=20.0).x).cuda()
flush = torch.empty(256 * 2**20, dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(1)
ctx = _native.context()
for b, loops in ((128, 8), (256, 8), (64, 8), (128, 4)):
    win = P.build_flat_window(n, b, 1e-8, delta_pass=1e-3)
    ps = [P.draw_permutation(n, rng) for _ in range(loops)]
    for _ in range(3):
        P.binned_spectrum(x, ps, win, b, precision=prec)
    tot = {}
    for _ in range(20):
        flush.zero_()
        torch.cuda.synchronize()
        ctx.set_profiling(True)
        P.binned_spectrum(x, ps, win, b, precision=prec)
        torch.cuda.synchronize()
        rep = ctx.profile_report()
        ctx.set_profiling(False)
        for k, v in rep.items():
            tot.setdefault(k, []).append(v[1] * 1e3)
    fold = {k: float(np.median(v)) for k, v in tot.items() if "fold" in k}
    print(f"{prec} B={b} loops={loops}: " + "  ".join(f"{k}={v:.1f}us" for k, v in fold.items())
          + (f"  ({134.2e6 / fold['k_fold_ml'] / 1e3:.0f} GB/s image)" if 'k_fold_ml' in fold else ""))
