"""SFFT (Algorithm 1, known k) timing: python tools/sfft_time.py [n] [k] [fp32|fp64]
(one transform at a time, CUDA events around 20 calls after warm-up, per-kernel profile)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prec = sys.argv[3] if len(sys.argv) > 3 else "fp32"
img = P.sparse_image(n, k, 7, snr_db=20.0)
x = torch.from_numpy(img.x).cuda()
cfg = P.SfftConfig(n=n, k=k)
for _ in range(3):
    out = P.sfft2d(x, cfg, 5, precision=prec)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    out = P.sfft2d(x, cfg, 5, precision=prec)
e1.record()
torch.cuda.synchronize()
print(f"sfft2d n={n} k={k} {prec}: {e0.elapsed_time(e1) / 20:.3f} ms per transform, {len(out)} coefficients, B={cfg.b_bins}")
ctx = _native.context(0)
ctx.set_profiling(True)
P.sfft2d(x, cfg, 5, precision=prec)
torch.cuda.synchronize()
rep = ctx.profile_report()
ctx.set_profiling(False)
for name, (cnt, ms, by) in sorted(rep.items(), key=lambda kv: -kv[1][1])[:10]:
    print(f"  {name:24s} {cnt:3d} launches {ms * 1e3:9.1f} us  {by / max(ms, 1e-9) / 1e6:8.1f} GB/s")
